// qforge_json.cpp -- the reference's JSON wire formats for circuits and Pauli
// sums (proj/src/circuit.cpp:524-571, proj/src/pauli.cpp:29-50) without a JSON
// library: a writer that produces what nlohmann::json::dump() produces for these
// documents (compact, keys sorted, shortest round-trip doubles with ".0" on
// integral values) and a small recursive-descent reader.  Errors follow the
// reference: malformed text or a missing key -> std::invalid_argument.
#include <charconv>
#include <cmath>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/pauli.hpp"

namespace qforge {
namespace {

// ---------------------------------------------------------------- writer
void put_double(std::string& s, double v) {
    if (!std::isfinite(v)) {  // nlohmann dumps non-finite numbers as null
        s += "null";
        return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    std::string t(buf, r.ptr);
    if (t.find_first_of(".eE") == std::string::npos) t += ".0";
    s += t;
}

template <class T> void put_int_array(std::string& s, const std::vector<T>& v) {
    s += '[';
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) s += ',';
        s += std::to_string(v[i]);
    }
    s += ']';
}

void put_double_array(std::string& s, const std::vector<double>& v) {
    s += '[';
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) s += ',';
        put_double(s, v[i]);
    }
    s += ']';
}

// ---------------------------------------------------------------- reader
struct Value {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    double num = 0;
    bool integral = false;
    std::string str;
    std::vector<Value> arr;
    std::map<std::string, Value> obj;

    const Value& at(const std::string& k) const {
        if (kind != Obj) throw std::invalid_argument("json: expected an object");
        auto it = obj.find(k);
        if (it == obj.end()) throw std::invalid_argument("json: missing key '" + k + "'");
        return it->second;
    }
    bool has(const std::string& k) const { return kind == Obj && obj.count(k); }
    double number() const {
        if (kind != Num) throw std::invalid_argument("json: expected a number");
        return num;
    }
    int integer() const {
        if (kind != Num || !integral) throw std::invalid_argument("json: expected an integer");
        return (int)num;
    }
    const std::vector<Value>& array() const {
        if (kind != Arr) throw std::invalid_argument("json: expected an array");
        return arr;
    }
    std::vector<int> ints() const {
        std::vector<int> out;
        for (const Value& v : array()) out.push_back(v.integer());
        return out;
    }
    std::vector<double> doubles() const {
        std::vector<double> out;
        for (const Value& v : array()) out.push_back(v.number());
        return out;
    }
};

struct Reader {
    const std::string& t;
    size_t i = 0;
    explicit Reader(const std::string& text) : t(text) {}

    [[noreturn]] void fail(const char* what) const {
        throw std::invalid_argument(std::string("json parse error: ") + what + " at offset " + std::to_string(i));
    }
    void ws() {
        while (i < t.size() && (t[i] == ' ' || t[i] == '\t' || t[i] == '\n' || t[i] == '\r')) ++i;
    }
    bool lit(const char* w) {
        const size_t n = std::char_traits<char>::length(w);
        if (t.compare(i, n, w) == 0) {
            i += n;
            return true;
        }
        return false;
    }
    std::string string() {
        if (i >= t.size() || t[i] != '"') fail("expected a string");
        ++i;
        std::string s;
        while (i < t.size() && t[i] != '"') {
            char c = t[i++];
            if (c == '\\') {
                if (i >= t.size()) fail("bad escape");
                const char e = t[i++];
                switch (e) {
                    case '"': case '\\': case '/': s += e; break;
                    case 'b': s += '\b'; break;
                    case 'f': s += '\f'; break;
                    case 'n': s += '\n'; break;
                    case 'r': s += '\r'; break;
                    case 't': s += '\t'; break;
                    case 'u': {  // keep ASCII code points (the wire formats use none)
                        if (i + 4 > t.size()) fail("bad \\u escape");
                        s += (char)std::stoi(t.substr(i, 4), nullptr, 16);
                        i += 4;
                        break;
                    }
                    default: fail("bad escape");
                }
            } else {
                s += c;
            }
        }
        if (i >= t.size()) fail("unterminated string");
        ++i;
        return s;
    }
    Value value() {
        ws();
        if (i >= t.size()) fail("unexpected end");
        Value v;
        const char c = t[i];
        if (c == '{') {
            ++i;
            v.kind = Value::Obj;
            ws();
            if (i < t.size() && t[i] == '}') {
                ++i;
                return v;
            }
            for (;;) {
                ws();
                std::string k = string();
                ws();
                if (i >= t.size() || t[i] != ':') fail("expected ':'");
                ++i;
                v.obj[k] = value();
                ws();
                if (i < t.size() && t[i] == ',') { ++i; continue; }
                if (i < t.size() && t[i] == '}') { ++i; break; }
                fail("expected ',' or '}'");
            }
        } else if (c == '[') {
            ++i;
            v.kind = Value::Arr;
            ws();
            if (i < t.size() && t[i] == ']') {
                ++i;
                return v;
            }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (i < t.size() && t[i] == ',') { ++i; continue; }
                if (i < t.size() && t[i] == ']') { ++i; break; }
                fail("expected ',' or ']'");
            }
        } else if (c == '"') {
            v.kind = Value::Str;
            v.str = string();
        } else if (lit("true")) {
            v.kind = Value::Bool;
            v.num = 1;
        } else if (lit("false")) {
            v.kind = Value::Bool;
        } else if (lit("null")) {
            v.kind = Value::Null;
        } else {
            const size_t b = i;
            while (i < t.size() && (std::isdigit((unsigned char)t[i]) || t[i] == '-' || t[i] == '+' || t[i] == '.' ||
                                    t[i] == 'e' || t[i] == 'E'))
                ++i;
            if (b == i) fail("unexpected character");
            double d = 0;
            auto r = std::from_chars(t.data() + b, t.data() + i, d);
            if (r.ec != std::errc() || r.ptr != t.data() + i) fail("bad number");
            v.kind = Value::Num;
            v.num = d;
            v.integral = t.find_first_of(".eE", b) >= i;
        }
        return v;
    }
    Value document() {
        Value v = value();
        ws();
        if (i != t.size()) fail("trailing characters");
        return v;
    }
};

}  // namespace

Gate gate_from_name(const std::string& s) {  // circuit.cpp:37-48
    static const std::pair<const char*, Gate> table[] = {
        {"h", Gate::h}, {"x", Gate::x}, {"y", Gate::y}, {"z", Gate::z}, {"s", Gate::s},
        {"rx", Gate::rx}, {"ry", Gate::ry}, {"rz", Gate::rz}, {"rzz", Gate::rzz},
        {"cx", Gate::cx}, {"cz", Gate::cz}, {"su4", Gate::su4}, {"csum", Gate::csum},
        {"subspace_ry", Gate::subspace_ry}, {"subspace_rz", Gate::subspace_rz}, {"unitary", Gate::unitary}};
    for (const auto& [name, g] : table)
        if (s == name) return g;
    throw std::invalid_argument("unknown gate name: " + s);
}

std::string Circuit::to_json() const {  // circuit.cpp:524-547
    std::string s = "{\"d\":" + std::to_string(d) + ",\"n\":" + std::to_string(n) + ",\"ops\":[";
    for (size_t k = 0; k < ops.size(); ++k) {
        const GateInstruction& op = ops[k];
        if (k) s += ',';
        s += '{';
        if (op.name == Gate::unitary) {  // keys in sorted order: im, name, params, re, rows, wires
            std::vector<double> im;
            for (std::int64_t r = 0; r < op.matrix.rows(); ++r)
                for (std::int64_t c = 0; c < op.matrix.cols(); ++c) im.push_back(op.matrix(r, c).imag());
            s += "\"im\":";
            put_double_array(s, im);
            s += ',';
        }
        s += "\"name\":\"" + gate_name(op.name) + "\",\"params\":";
        put_double_array(s, op.params);
        if (op.name == Gate::unitary) {
            std::vector<double> re;
            for (std::int64_t r = 0; r < op.matrix.rows(); ++r)
                for (std::int64_t c = 0; c < op.matrix.cols(); ++c) re.push_back(op.matrix(r, c).real());
            s += ",\"re\":";
            put_double_array(s, re);
            s += ",\"rows\":" + std::to_string(op.matrix.rows());
        }
        s += ",\"wires\":";
        put_int_array(s, op.wires);
        s += '}';
    }
    s += "]}";
    return s;
}

Circuit Circuit::from_json(const std::string& text) {  // circuit.cpp:549-571
    const Value j = Reader(text).document();
    Circuit c(j.at("n").integer(), j.has("d") ? j.at("d").integer() : 2);
    for (const Value& o : j.at("ops").array()) {
        const Value& nm = o.at("name");
        if (nm.kind != Value::Str) throw std::invalid_argument("json: gate name must be a string");
        const Gate g = gate_from_name(nm.str);
        std::vector<int> wires = o.at("wires").ints();
        std::vector<double> params = o.at("params").doubles();
        if (g == Gate::unitary) {
            const int rows = o.at("rows").integer();
            const std::vector<double> re = o.at("re").doubles(), im = o.at("im").doubles();
            if ((int)re.size() < rows * rows || (int)im.size() < rows * rows)
                throw std::invalid_argument("json: unitary matrix entries missing");
            ComplexMatrix m(rows, rows);
            for (int r = 0; r < rows; ++r)
                for (int col = 0; col < rows; ++col) m(r, col) = cplx(re[r * rows + col], im[r * rows + col]);
            c.unitary(wires, m);
        } else {
            c.gate(g, wires, params);
        }
    }
    return c;
}

std::string PauliSum::to_json() const {  // pauli.cpp:29-39
    std::string s = "{\"n\":" + std::to_string(n) + ",\"terms\":[";
    for (size_t k = 0; k < terms.size(); ++k) {
        if (k) s += ',';
        s += "{\"codes\":";
        put_int_array(s, terms[k].codes);
        s += ",\"w_im\":";
        put_double(s, terms[k].weight.imag());
        s += ",\"w_re\":";
        put_double(s, terms[k].weight.real());
        s += '}';
    }
    s += "]}";
    return s;
}

PauliSum PauliSum::from_json(const std::string& text) {  // pauli.cpp:41-50
    const Value j = Reader(text).document();
    PauliSum h;
    h.n = j.at("n").integer();
    for (const Value& t : j.at("terms").array())
        h.add(cplx(t.at("w_re").number(), t.at("w_im").number()), t.at("codes").ints());
    return h;
}

}  // namespace qforge
