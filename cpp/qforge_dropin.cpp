// qforge_dropin.cpp -- the reference qforge hot-path API (include/qforge/*.hpp)
// implemented over the C-ABI of the B200 engine (include/qforge_b200.h).
// Host-only C++: validation and exceptions follow the reference
// (require() -> std::invalid_argument); every state-vector operation runs on
// the GPU through libqforge_b200.so.  Reference line citations are relative to
// /root/reference/proj.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "qforge/circuit.hpp"
#include "qforge/lattice.hpp"
#include "qforge/noise.hpp"
#include "qforge/shadows.hpp"
#include "qforge/pauli.hpp"
#include "qforge/variational.hpp"
#include "qforge_b200.h"

namespace qforge {

// ------------------------------------------------------------------ engine glue
namespace {

Precision g_prec = Precision::c128;
std::mutex g_mu;

void check(int rc) {
    if (rc == QF_OK) return;
    const std::string msg = qf_last_error();
    if (rc == QF_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

qf_ctx* ctx() {
    static qf_ctx* c = nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    if (!c) {
        const char* e = std::getenv("QF_DEVICE");
        check(qf_ctx_create(e ? std::atoi(e) : 0, &c));
    }
    return c;
}

struct ProgramHandle {
    qf_program* p = nullptr;
    ~ProgramHandle() {
        if (p) qf_program_destroy(p);
    }
};

struct ObservableHandle {
    qf_observable* o = nullptr;
    ~ObservableHandle() {
        if (o) qf_observable_destroy(o);
    }
};

struct Template {
    int n = 0;
    std::vector<qf_op> ops;
    std::vector<double> mats;  // [n_mats][4][4][2]
    std::optional<ComplexVector> init;
};

void push_matrix(std::vector<double>& mats, const ComplexMatrix& m) {
    const int d = (int)m.rows();
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            const cplx v = (r < d && c < d) ? m(r, c) : cplx(0.0);
            mats.push_back(v.real());
            mats.push_back(v.imag());
        }
}

bool is_rotation(Gate g) { return g == Gate::rx || g == Gate::ry || g == Gate::rz || g == Gate::rzz; }

// Circuit -> qf ops; slot_of[i] = {slot, coef, offset} for rotations fed by theta
struct SlotMap {
    int slot = -1;
    double coef = 1.0, offset = 0.0;
};
Template circuit_template(const Circuit& c, const std::vector<SlotMap>* slots) {
    require(c.d == 2, "device path: qubit circuits only (d == 2)");
    Template t;
    t.n = c.n;
    t.init = c.initial_state;
    for (size_t i = 0; i < c.ops.size(); ++i) {
        const GateInstruction& op = c.ops[i];
        qf_op q{};
        q.kind = (int)op.name;
        q.q0 = op.wires.at(0);
        q.q1 = op.wires.size() > 1 ? op.wires[1] : -1;
        q.slot = -1;
        q.coef = 1.0;
        q.offset = 0.0;
        q.mat = -1;
        if (op.name == Gate::su4 || op.name == Gate::unitary) {
            push_matrix(t.mats, gate_matrix(op, 2));
            q.mat = (int)(t.mats.size() / 32) - 1;
        } else if (is_rotation(op.name)) {
            if (slots && (*slots)[i].slot >= 0) {
                q.slot = (*slots)[i].slot;
                q.coef = (*slots)[i].coef;
                q.offset = (*slots)[i].offset;
            } else {
                q.offset = op.params.at(0);
            }
        } else if (op.name == Gate::csum || op.name == Gate::subspace_ry || op.name == Gate::subspace_rz) {
            throw std::invalid_argument("gate_matrix: qudit gates are not supported on the qubit device path");
        }
        t.ops.push_back(q);
    }
    return t;
}

std::shared_ptr<ProgramHandle> make_program(const Template& t, int n_params) {
    auto h = std::make_shared<ProgramHandle>();
    check(qf_program_create(ctx(), t.n, (int)t.ops.size(), t.ops.data(), t.mats.empty() ? nullptr : t.mats.data(),
                            (int)(t.mats.size() / 32), n_params, (int)g_prec, &h->p));
    if (t.init) {
        require(t.init->size() == (std::int64_t)1 << t.n, "run: initial state size mismatch");
        check(qf_program_set_initial_state(h->p, reinterpret_cast<const double*>(t.init->data())));
    }
    return h;
}

// FNV-1a over raw bytes (device-cache keys: content, not identity or size)
struct Fnv {
    std::uint64_t h = 1469598103934665603ull;
    void add(const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) {
            h ^= b[i];
            h *= 1099511628211ull;
        }
    }
    template <class T> void add(const T& v) { add(&v, sizeof v); }
};

std::uint64_t pauli_sum_key(const PauliSum& h) {
    Fnv f;
    f.add(h.n);
    f.add(h.terms.size());
    for (const auto& t : h.terms) {
        f.add(t.weight);
        f.add(t.codes.size());
        for (int c : t.codes) f.add(c);
    }
    return f.h;
}

qf_observable* observable(const PauliSum& h) {
    // keyed on the sum's content: `terms` is public and may be edited in place,
    // and a copied PauliSum shares the cache pointer until it diverges
    struct Cache {
        std::shared_ptr<ObservableHandle> obs;
        std::uint64_t key = 0;
    };
    const std::uint64_t key = pauli_sum_key(h);
    auto cache = std::static_pointer_cast<Cache>(h.device_cache);
    if (!cache || cache->key != key) {
        cache = std::make_shared<Cache>();
        std::vector<int8_t> codes;
        std::vector<double> wr, wi;
        for (const auto& t : h.terms) {
            for (int c : t.codes) codes.push_back((int8_t)c);
            wr.push_back(t.weight.real());
            wi.push_back(t.weight.imag());
        }
        cache->obs = std::make_shared<ObservableHandle>();
        check(qf_observable_create(ctx(), h.n, (int)h.terms.size(), codes.data(), wr.data(), wi.data(),
                                   &cache->obs->o));
        cache->key = key;
        h.device_cache = cache;
    }
    return cache->obs->o;
}

// 4x4 (or 2x2) complex matrix exponential: scaling and squaring + Taylor
ComplexMatrix expm_small(const ComplexMatrix& a) {
    const int d = (int)a.rows();
    double nrm = 0;
    for (int r = 0; r < d; ++r) {
        double s = 0;
        for (int c = 0; c < d; ++c) s += std::abs(a(r, c));
        nrm = std::max(nrm, s);
    }
    int sq = std::max(0, (int)std::ceil(std::log2(std::max(nrm, 1e-300))) + 1);
    ComplexMatrix b = a * cplx(std::ldexp(1.0, -sq));
    ComplexMatrix res = ComplexMatrix::Identity(d, d), term = ComplexMatrix::Identity(d, d);
    for (int k = 1; k <= 20; ++k) {
        term = term * b * cplx(1.0 / k);
        res = res + term;
    }
    for (int i = 0; i < sq; ++i) res = res * res;
    return res;
}

}  // namespace

void set_device_precision(Precision p) { g_prec = p; }
Precision device_precision() { return g_prec; }

// ------------------------------------------------------------------ circuits
std::string gate_name(Gate g) {
    static const char* names[] = {"h", "x", "y", "z", "s", "rx", "ry", "rz", "rzz", "cx", "cz", "su4",
                                  "csum", "subspace_ry", "subspace_rz", "unitary"};
    const int i = (int)g;
    return (i >= 0 && i < 16) ? names[i] : "?";
}

StateVector StateVector::zero_state(int n, int d) {  // circuit.cpp:69-76
    StateVector psi;
    psi.n = n;
    psi.d = d;
    std::int64_t dim = 1;
    for (int i = 0; i < n; ++i) dim *= d;
    psi.amps = ComplexVector::Zero(dim);
    psi.amps[0] = 1.0;
    return psi;
}

Circuit& Circuit::gate(Gate g, std::vector<int> wires, std::vector<double> params) {  // circuit.cpp:178-186
    for (int w : wires) require(w >= 0 && w < n, "Circuit: wire out of range");
    for (size_t a = 0; a < wires.size(); ++a)
        for (size_t b = a + 1; b < wires.size(); ++b) require(wires[a] != wires[b], "Circuit: duplicate wires");
    for (double p : params) require(std::isfinite(p), "Circuit: non-finite parameter");
    ops.push_back({g, std::move(wires), std::move(params), {}});
    return *this;
}

Circuit& Circuit::su4(int a, int b, const std::vector<double>& theta) {  // circuit.cpp:188-191
    require(theta.size() == 15, "su4: needs 15 parameters");
    return gate(Gate::su4, {a, b}, theta);
}

Circuit& Circuit::unitary(std::vector<int> wires, const ComplexMatrix& u) {  // circuit.cpp:193-200
    ComplexMatrix check_m = u.adjoint() * u;
    require((check_m - ComplexMatrix::Identity(u.rows(), u.cols())).cwiseAbs().maxCoeff() < 1e-10,
            "unitary: matrix is not unitary");
    gate(Gate::unitary, wires, {});
    ops.back().matrix = u;
    return *this;
}

ComplexMatrix gate_matrix(const GateInstruction& instr, int d) {  // circuit.cpp:202-302 (qubit gates)
    require(d == 2, "gate_matrix: qubit-only gate in a qudit circuit");
    const double isq = 1.0 / std::sqrt(2.0);
    const cplx I(0.0, 1.0);
    auto m2 = [](cplx a, cplx b, cplx c, cplx e) { return (ComplexMatrix(2, 2) << a, b, c, e).finished(); };
    switch (instr.name) {
        case Gate::h: return m2(isq, isq, isq, -isq);
        case Gate::x: return m2(0, 1, 1, 0);
        case Gate::y: return m2(0, -I, I, 0);
        case Gate::z: return m2(1, 0, 0, -1);
        case Gate::s: return m2(1, 0, 0, I);
        case Gate::rx: {
            const double t = instr.params.at(0);
            const cplx c = std::cos(0.5 * t), s = cplx(0.0, -std::sin(0.5 * t));
            return m2(c, s, s, c);
        }
        case Gate::ry: {
            const double t = instr.params.at(0), c = std::cos(0.5 * t), s = std::sin(0.5 * t);
            return m2(c, -s, s, c);
        }
        case Gate::rz: {
            const double t = instr.params.at(0);
            return m2(std::polar(1.0, -0.5 * t), 0, 0, std::polar(1.0, 0.5 * t));
        }
        case Gate::rzz: {
            const double t = instr.params.at(0);
            ComplexMatrix m = ComplexMatrix::Zero(4, 4);
            const cplx em = std::polar(1.0, -0.5 * t), ep = std::polar(1.0, 0.5 * t);
            m(0, 0) = em; m(1, 1) = ep; m(2, 2) = ep; m(3, 3) = em;
            return m;
        }
        case Gate::cx: {
            ComplexMatrix m = ComplexMatrix::Zero(4, 4);
            m(0, 0) = m(1, 1) = m(2, 3) = m(3, 2) = 1.0;
            return m;
        }
        case Gate::cz: {
            ComplexMatrix m = ComplexMatrix::Identity(4, 4);
            m(3, 3) = -1.0;
            return m;
        }
        case Gate::su4: {  // exp(-i/2 sum theta_k P_k), lexicographic words without (0,0)
            require(instr.params.size() == 15, "su4: needs 15 parameters");
            const ComplexMatrix single[4] = {ComplexMatrix::Identity(2, 2), m2(0, 1, 1, 0), m2(0, -I, I, 0),
                                             m2(1, 0, 0, -1)};
            ComplexMatrix gen = ComplexMatrix::Zero(4, 4);
            int k = 0;
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) {
                    if (a == 0 && b == 0) continue;
                    for (int r = 0; r < 4; ++r)
                        for (int c = 0; c < 4; ++c)
                            gen(r, c) += instr.params[k] * single[a](r >> 1, c >> 1) * single[b](r & 1, c & 1);
                    ++k;
                }
            return expm_small(gen * cplx(0.0, -0.5));
        }
        case Gate::unitary: return instr.matrix;
        default: break;
    }
    throw std::invalid_argument("gate_matrix: qudit gates are not supported on the qubit device path");
}

StateVector run(const Circuit& c, std::size_t memory_guard_log2) {  // circuit.cpp:304-317
    require(std::pow((double)c.d, c.n) <= std::pow(2.0, (double)memory_guard_log2),
            "run: state dimension exceeds memory guard");
    Template t = circuit_template(c, nullptr);
    auto prog = make_program(t, 0);
    StateVector psi;
    psi.n = c.n;
    psi.d = c.d;
    psi.amps = ComplexVector::Zero((std::int64_t)1 << c.n);
    check(qf_run_state(ctx(), prog->p, nullptr, (int)memory_guard_log2, reinterpret_cast<double*>(psi.amps.data())));
    return psi;
}

void apply_local_unitary(StateVector& psi, const ComplexMatrix& u, const std::vector<int>& wires) {
    const int k = (int)wires.size();
    require(u.rows() == ((std::int64_t)1 << k) && u.cols() == ((std::int64_t)1 << k),
            "apply_local_unitary: wrong gate size");
    for (int w : wires) require(w >= 0 && w < psi.n, "apply_local_unitary: wire out of range");
    std::vector<double> um;  // row-major for the C-ABI (ComplexMatrix is column-major, like Eigen)
    um.reserve((size_t)u.size() * 2);
    for (std::int64_t r = 0; r < u.rows(); ++r)
        for (std::int64_t c = 0; c < u.cols(); ++c) {
            um.push_back(u(r, c).real());
            um.push_back(u(r, c).imag());
        }
    check(qf_apply_unitary(ctx(), psi.n, reinterpret_cast<double*>(psi.amps.data()), k, wires.data(), um.data()));
}

cplx expectation_pauli(const StateVector& psi, const PauliSum& obs) {  // circuit.cpp:319-347
    require(psi.d == 2, "expectation_pauli: qubits only");
    require(obs.n == psi.n, "expectation_pauli: size mismatch");
    Circuit c(psi.n);
    c.initial_state = psi.amps;
    auto prog = make_program(circuit_template(c, nullptr), 0);
    double out[2];
    check(qf_expectation(ctx(), prog->p, observable(obs), nullptr, out));
    return cplx(out[0], out[1]);
}

// ------------------------------------------------------------------ lattice / Pauli sums
Lattice build_lattice(LatticeKind kind, const std::vector<int>& size, const std::vector<bool>& pbc,
                      double lattice_constant, int neighbor_order) {  // lattice.cpp:89-170 (chain)
    require(kind == LatticeKind::chain, "build_lattice: only the chain lattice is on the device hot path");
    require(lattice_constant > 0.0, "build_lattice: lattice_constant must be > 0");
    require(size.size() == 1 && pbc.size() == 1, "build_lattice: wrong size rank");
    const int n = size[0];
    require(n >= 1, "build_lattice: size entries must be >= 1");
    if (pbc[0]) require(n >= 3, "build_lattice: periodic dimension needs extent >= 3");
    Lattice l;
    l.kind = kind;
    l.lattice_constant = lattice_constant;
    l.n_sites = n;
    struct P { double d; int i, j; };
    std::vector<P> pairs;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            double d = std::abs((double)(i - j)) * lattice_constant;
            if (pbc[0])
                for (int m = -1; m <= 1; ++m) d = std::min(d, std::abs((double)(i - j + m * n)) * lattice_constant);
            pairs.push_back({d, i, j});
        }
    std::sort(pairs.begin(), pairs.end(), [](const P& a, const P& b) {
        if (a.d != b.d) return a.d < b.d;
        if (a.i != b.i) return a.i < b.i;
        return a.j < b.j;
    });
    int order = 0;
    double shell = -1.0;
    for (const P& p : pairs) {
        if (p.d <= 0.0) continue;
        if (shell < 0.0 || p.d > shell * (1.0 + 1e-6)) {
            ++order;
            shell = p.d;
        }
        if (order > neighbor_order) break;
        l.edges_by_order[order].push_back({p.i, p.j});
    }
    return l;
}

void PauliSum::add(cplx weight, const std::vector<int>& codes) {  // pauli.cpp:12-18
    require(static_cast<int>(codes.size()) == n, "PauliSum::add: wrong code length");
    for (int c : codes) require(c >= 0 && c <= 3, "PauliSum::add: code out of range");
    require(std::isfinite(weight.real()) && std::isfinite(weight.imag()), "PauliSum::add: non-finite weight");
    terms.push_back({weight, codes});
}

void PauliSum::add_word(cplx weight, const std::vector<std::pair<int, int>>& site_codes) {  // pauli.cpp:20-27
    std::vector<int> codes(n, 0);
    for (const auto& [site, code] : site_codes) {
        require(site >= 0 && site < n, "PauliSum::add_word: site out of range");
        codes[site] = code;
    }
    add(weight, codes);
}

PauliSum tfim_terms(const Lattice& l, double g) {  // pauli.cpp:181-189
    PauliSum h;
    h.n = static_cast<int>(l.num_sites());
    auto it = l.edges_by_order.find(1);
    require(it != l.edges_by_order.end(), "tfim_terms: lattice has no order-1 edges");
    for (const auto& [i, j] : it->second) h.add_word(-1.0, {{i, 3}, {j, 3}});
    for (int i = 0; i < h.n; ++i) h.add_word(-g, {{i, 1}});
    return h;
}

PauliSum heisenberg_terms(const Lattice& l, double jx, double jy, double jz) {  // pauli.cpp:191-203
    PauliSum h;
    h.n = static_cast<int>(l.num_sites());
    auto it = l.edges_by_order.find(1);
    require(it != l.edges_by_order.end(), "heisenberg_terms: lattice has no order-1 edges");
    const double js[3] = {jx, jy, jz};
    for (const auto& [i, j] : it->second)
        for (int axis = 0; axis < 3; ++axis)
            if (js[axis] != 0.0) h.add_word(js[axis], {{i, axis + 1}, {j, axis + 1}});
    return h;
}

// ------------------------------------------------------------------ sparse
SparseCOO pauli_sum_to_coo(const PauliSum& h, int n_guard, std::size_t /*workers*/) {  // pauli.cpp:89-153
    require(h.n >= 1, "pauli_sum_to_coo: empty system");
    require(h.n <= n_guard, "pauli_sum_to_coo: qubit count exceeds memory guard");
    SparseCOO out;
    out.dim = (std::int64_t)1 << h.n;
    std::int64_t nnz = 0;
    check(qf_pauli_sum_to_coo(ctx(), observable(h), n_guard, 0, nullptr, nullptr, nullptr, 0, &nnz));
    out.rows.resize((size_t)nnz);
    out.cols.resize((size_t)nnz);
    out.vals.resize((size_t)nnz);
    if (nnz)
        check(qf_pauli_sum_to_coo(ctx(), observable(h), n_guard, 0, out.rows.data(), out.cols.data(),
                                  reinterpret_cast<double*>(out.vals.data()), nnz, &nnz));
    return out;
}

void SparseCOO::canonicalize() {  // sparse.hpp:25 contract
    std::vector<size_t> idx(vals.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
        return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
    });
    SparseCOO c;
    c.dim = dim;
    for (size_t i : idx) {
        if (!c.vals.empty() && c.rows.back() == rows[i] && c.cols.back() == cols[i]) c.vals.back() += vals[i];
        else c.push(rows[i], cols[i], vals[i]);
    }
    SparseCOO z;
    z.dim = dim;
    for (size_t k = 0; k < c.vals.size(); ++k)
        if (c.vals[k] != cplx(0.0)) z.push(c.rows[k], c.cols[k], c.vals[k]);
    *this = std::move(z);
}

void SparseCOO::matvec(const ComplexVector& in, ComplexVector& out) const {
    require(in.size() == dim, "SparseCOO::matvec: size mismatch");
    out = ComplexVector::Zero(dim);
    for (size_t k = 0; k < vals.size(); ++k) out[rows[k]] += vals[k] * in[cols[k]];
}

ComplexVector SparseCOO::apply(const ComplexVector& in) const {
    ComplexVector out;
    matvec(in, out);
    return out;
}

ComplexMatrix SparseCOO::to_dense() const {
    ComplexMatrix m = ComplexMatrix::Zero(dim, dim);
    for (size_t k = 0; k < vals.size(); ++k) m(rows[k], cols[k]) += vals[k];
    return m;
}

SparseCOO SparseCOO::from_dense(const ComplexMatrix& m) {
    require(m.rows() == m.cols(), "SparseCOO::from_dense: matrix must be square");
    SparseCOO s;
    s.dim = m.rows();
    for (std::int64_t r = 0; r < m.rows(); ++r)
        for (std::int64_t c = 0; c < m.cols(); ++c)
            if (m(r, c) != cplx(0.0)) s.push(r, c, m(r, c));
    return s;
}

SparseCOO SparseCOO::operator+(const SparseCOO& other) const {
    require(dim == other.dim, "SparseCOO::operator+: dimension mismatch");
    SparseCOO s = *this;
    for (size_t k = 0; k < other.vals.size(); ++k) s.push(other.rows[k], other.cols[k], other.vals[k]);
    s.canonicalize();
    return s;
}

// ------------------------------------------------------------------ shadows (shadows.cpp)
void ShadowDataset::validate() const {
    require(n >= 1, "ShadowDataset: n must be >= 1");
    require(bases.size() == outcomes.size(), "ShadowDataset: row count mismatch");
    for (size_t r = 0; r < bases.size(); ++r) {
        require((int)bases[r].size() == n, "ShadowDataset: bad basis row");
        require((int)outcomes[r].size() == n, "ShadowDataset: bad outcome row");
        for (int c : bases[r]) require(c >= 1 && c <= 3, "ShadowDataset: bad basis code");
        for (int b : outcomes[r]) require(b == 0 || b == 1, "ShadowDataset: bad outcome");
    }
}

std::vector<std::vector<int>> random_bases(std::size_t m, int n, RngStream& rng) {  // shadows.cpp:24-29
    std::vector<std::vector<int>> out(m, std::vector<int>(n));
    for (auto& row : out)
        for (int& c : row) c = 1 + (int)rng.uniform_below(3);
    return out;
}

ShadowDataset shadow_snapshots(const StateVector& psi, const std::vector<std::vector<int>>& bases, RngStream& rng,
                               int /*workers*/) {  // shadows.cpp:50-85
    require(psi.d == 2, "shadow_snapshots: qubits only");
    const size_t m = bases.size();
    ShadowDataset ds;
    ds.n = psi.n;
    ds.bases = bases;
    ds.outcomes.assign(m, std::vector<int>(psi.n, 0));
    if (m == 0) return ds;
    std::vector<int8_t> codes(m * psi.n);
    for (size_t r = 0; r < m; ++r) {
        require((int)bases[r].size() == psi.n, "shadow_snapshots: bad basis row");
        for (int q = 0; q < psi.n; ++q) codes[r * psi.n + q] = (int8_t)bases[r][q];
    }
    const std::vector<RngStream> streams = rng.split(m);
    std::vector<double> u(m);
    for (size_t r = 0; r < m; ++r) u[r] = RngStream(streams[r]).uniform();
    Circuit c(psi.n);
    c.initial_state = psi.amps;
    auto prog = make_program(circuit_template(c, nullptr), 0);
    std::vector<int8_t> out(m * psi.n);
    check(qf_shadow_snapshots(ctx(), prog->p, nullptr, (int)m, codes.data(), u.data(), out.data()));
    for (size_t r = 0; r < m; ++r)
        for (int q = 0; q < psi.n; ++q) ds.outcomes[r][q] = out[r * psi.n + q];
    return ds;
}

double estimate_pauli(const ShadowDataset& ds, const std::vector<int>& obs_codes, int n_batches) {  // :86-122
    require((int)obs_codes.size() == ds.n, "estimate_pauli: length mismatch");
    require(n_batches >= 1, "estimate_pauli: n_batches must be >= 1");
    std::vector<int> support;
    for (int q = 0; q < ds.n; ++q) {
        require(obs_codes[q] >= 0 && obs_codes[q] <= 3, "estimate_pauli: bad code");
        if (obs_codes[q]) support.push_back(q);
    }
    if (support.empty()) return 1.0;
    const size_t m = ds.size();
    require(m > 0, "estimate_pauli: empty dataset");
    require((size_t)n_batches <= m, "estimate_pauli: more batches than snapshots");
    std::vector<double> mean(n_batches, 0.0);
    std::vector<size_t> cnt(n_batches, 0);
    for (size_t r = 0; r < m; ++r) {
        double v = 1.0;
        for (int q : support) {
            if (ds.bases[r][q] != obs_codes[q]) {
                v = 0.0;
                break;
            }
            v *= 3.0 * (1.0 - 2.0 * ds.outcomes[r][q]);
        }
        const size_t b = r * n_batches / m;
        mean[b] += v;
        ++cnt[b];
    }
    for (int b = 0; b < n_batches; ++b) mean[b] /= (double)cnt[b];
    std::sort(mean.begin(), mean.end());
    return n_batches % 2 ? mean[n_batches / 2] : 0.5 * (mean[n_batches / 2 - 1] + mean[n_batches / 2]);
}

void save_dataset(const ShadowDataset& ds, const std::string& path) {  // :124-136
    ds.validate();
    std::ofstream f(path);
    require(f.good(), ("save_dataset: cannot open " + path).c_str());
    f << ds.n << "," << ds.size() << "\n";
    for (size_t r = 0; r < ds.size(); ++r) {
        for (int c : ds.bases[r]) f << c;
        f << ";";
        for (int b : ds.outcomes[r]) f << b;
        f << "\n";
    }
    require(f.good(), "save_dataset: write failed");
}

ShadowDataset load_dataset(const std::string& path) {  // :138-170
    std::ifstream f(path);
    require(f.good(), ("load_dataset: cannot open " + path).c_str());
    std::string line;
    require((bool)std::getline(f, line), "load_dataset: missing header");
    const size_t comma = line.find(',');
    require(comma != std::string::npos, "load_dataset: bad header");
    ShadowDataset ds;
    ds.n = std::stoi(line.substr(0, comma));
    const size_t m = std::stoul(line.substr(comma + 1));
    while (std::getline(f, line)) {
        if (line.empty()) continue;
        const size_t semi = line.find(';');
        require(semi != std::string::npos, "load_dataset: bad row");
        const std::string bs = line.substr(0, semi), os = line.substr(semi + 1);
        require(bs.size() == (size_t)ds.n && os.size() == bs.size(), "load_dataset: bad row length");
        std::vector<int> br(ds.n), orow(ds.n);
        for (int q = 0; q < ds.n; ++q) {
            br[q] = bs[q] - '0';
            orow[q] = os[q] - '0';
        }
        ds.bases.push_back(br);
        ds.outcomes.push_back(orow);
    }
    require(ds.size() == m, "load_dataset: row count mismatch");
    ds.validate();
    return ds;
}

// ------------------------------------------------------------------ noise (noise.cpp)
double KrausChannel::completeness_defect() const {
    if (operators.empty()) return 1.0;
    const std::int64_t d = operators.front().rows();
    ComplexMatrix acc = ComplexMatrix::Zero(d, d);
    for (const auto& k : operators) acc = acc + k.adjoint() * k;
    return (acc - ComplexMatrix::Identity(d, d)).cwiseAbs().maxCoeff();
}

void KrausChannel::validate() const {
    require(!operators.empty(), "KrausChannel: no operators");
    const std::int64_t d = (std::int64_t)1 << arity;
    for (const auto& k : operators) require(k.rows() == d && k.cols() == d, "KrausChannel: wrong operator shape");
    require(completeness_defect() <= 1e-10, "KrausChannel: completeness violated");
}

namespace {
ComplexMatrix mat2(cplx a, cplx b, cplx c, cplx d) { return (ComplexMatrix(2, 2) << a, b, c, d).finished(); }
ComplexMatrix kron(const ComplexMatrix& a, const ComplexMatrix& b) {
    ComplexMatrix o(a.rows() * b.rows(), a.cols() * b.cols());
    for (std::int64_t i = 0; i < a.rows(); ++i)
        for (std::int64_t j = 0; j < a.cols(); ++j)
            for (std::int64_t k = 0; k < b.rows(); ++k)
                for (std::int64_t l = 0; l < b.cols(); ++l) o(i * b.rows() + k, j * b.cols() + l) = a(i, j) * b(k, l);
    return o;
}
}  // namespace

KrausChannel depolarizing_channel(double p, int k) {  // noise.cpp:27-60
    require(p >= 0.0 && p <= 1.0, "depolarizing_channel: p out of range");
    require(k >= 1 && k <= 3, "depolarizing_channel: arity out of range");
    const cplx I(0.0, 1.0);
    const ComplexMatrix paulis[4] = {ComplexMatrix::Identity(2, 2), mat2(0, 1, 1, 0), mat2(0, -I, I, 0), mat2(1, 0, 0, -1)};
    KrausChannel ch;
    ch.name = "depolarizing";
    ch.arity = k;
    int words = 1;
    for (int i = 0; i < k; ++i) words *= 4;
    const double pw = p / (words - 1);
    for (int w = 0; w < words; ++w) {
        const double weight = w == 0 ? 1.0 - p : pw;
        if (weight == 0.0) continue;
        ComplexMatrix op = ComplexMatrix::Identity(1, 1);
        for (int site = 0, ww = w; site < k; ++site, ww /= 4) op = kron(paulis[ww % 4], op);
        ch.operators.push_back(op * cplx(std::sqrt(weight)));
    }
    ch.validate();
    return ch;
}

KrausChannel amplitude_damping_channel(double gamma) {  // noise.cpp:62-72
    require(gamma >= 0.0 && gamma <= 1.0, "amplitude_damping_channel: gamma out of range");
    KrausChannel ch{"amplitude_damping", 1, {mat2(1, 0, 0, std::sqrt(1.0 - gamma)), mat2(0, std::sqrt(gamma), 0, 0)}};
    ch.validate();
    return ch;
}

KrausChannel phase_damping_channel(double lambda) {  // noise.cpp:74-84
    require(lambda >= 0.0 && lambda <= 1.0, "phase_damping_channel: lambda out of range");
    KrausChannel ch{"phase_damping", 1, {mat2(1, 0, 0, std::sqrt(1.0 - lambda)), mat2(0, 0, 0, std::sqrt(lambda))}};
    ch.validate();
    return ch;
}

KrausChannel reset_channel(double p) {  // noise.cpp:86-97
    require(p >= 0.0 && p <= 1.0, "reset_channel: p out of range");
    const double sp = std::sqrt(p), sq = std::sqrt(1.0 - p);
    KrausChannel ch{"reset", 1, {mat2(sq, 0, 0, sq), mat2(sp, 0, 0, 0), mat2(0, sp, 0, 0)}};
    ch.validate();
    return ch;
}

KrausChannel thermal_relaxation_channel(double gamma, double lambda) {  // noise.cpp:99-111
    const KrausChannel ad = amplitude_damping_channel(gamma), pd = phase_damping_channel(lambda);
    KrausChannel ch;
    ch.name = "thermal_relaxation";
    ch.arity = 1;
    for (const auto& k2 : pd.operators)
        for (const auto& k1 : ad.operators) ch.operators.push_back(k2 * k1);
    ch.validate();
    return ch;
}

void NoiseConf::attach(const std::string& gate, KrausChannel channel) {  // noise.cpp:113-131
    channel.validate();
    rules.push_back({gate, std::nullopt, nullptr, std::move(channel)});
}

void NoiseConf::attach_on_wires(const std::string& gate, std::vector<int> wires, KrausChannel channel) {
    channel.validate();
    require(channel.arity == (int)wires.size(), "NoiseConf: channel arity does not match wire tuple");
    rules.push_back({gate, std::move(wires), nullptr, std::move(channel)});
}

void NoiseConf::attach_predicate(std::function<bool(const GateInstruction&)> pred, KrausChannel channel) {
    channel.validate();
    rules.push_back({"", std::nullopt, std::move(pred), std::move(channel)});
}

std::vector<const KrausChannel*> NoiseConf::match(const GateInstruction& instr) const {  // noise.cpp:133-145
    std::vector<const KrausChannel*> out;
    for (const auto& r : rules) {
        if (!r.gate.empty() && r.gate != gate_name(instr.name)) continue;
        if (r.wires && *r.wires != instr.wires) continue;
        if (r.predicate && !r.predicate(instr)) continue;
        if (r.channel.arity != (int)instr.wires.size()) continue;
        out.push_back(&r.channel);
    }
    return out;
}

std::vector<Trajectory> mc_trajectories(const Circuit& c, const NoiseConf& conf, RngStream& rng, int count) {
    require(c.d == 2, "mc_trajectory: qubits only");
    require(count >= 0, "mc_trajectories: negative count");
    Template t = circuit_template(c, nullptr);
    std::vector<int> ptr{0}, ids, kptr{0};
    std::vector<double> kraus;
    std::vector<const KrausChannel*> chans;
    for (const auto& instr : c.ops) {
        for (const KrausChannel* ch : conf.match(instr)) {
            auto it = std::find(chans.begin(), chans.end(), ch);
            if (it == chans.end()) {
                chans.push_back(ch);
                for (const auto& k : ch->operators) push_matrix(kraus, k);
                kptr.push_back((int)(kraus.size() / 32));
                it = chans.end() - 1;
            }
            ids.push_back((int)(it - chans.begin()));
        }
        ptr.push_back((int)ids.size());
    }
    const int n_apps = (int)ids.size();
    std::vector<double> u((size_t)count * n_apps);
    for (auto& x : u) x = rng.uniform();  // the reference draws one uniform per application, in order
    const size_t N = (size_t)1 << c.n;
    std::vector<cplx> states((size_t)count * N);
    std::vector<double> logp(count);
    if (count > 0)
        check(qf_noise_trajectories(ctx(), c.n, (int)t.ops.size(), t.ops.data(), t.mats.empty() ? nullptr : t.mats.data(),
                                    (int)(t.mats.size() / 32), ptr.data(), ids.data(), kptr.data(),
                                    kraus.empty() ? nullptr : kraus.data(),
                                    t.init ? reinterpret_cast<const double*>(t.init->data()) : nullptr, count,
                                    u.empty() ? nullptr : u.data(), (int)g_prec,
                                    reinterpret_cast<double*>(states.data()), logp.data(), nullptr, nullptr));
    std::vector<Trajectory> out(count);
    for (int k = 0; k < count; ++k) {
        out[k].state.n = c.n;
        out[k].state.d = 2;
        out[k].state.amps = ComplexVector::Zero((std::int64_t)N);
        std::copy(states.begin() + (size_t)k * N, states.begin() + (size_t)(k + 1) * N, out[k].state.amps.data());
        out[k].log_prob = logp[k];
    }
    return out;
}

Trajectory mc_trajectory(const Circuit& c, const NoiseConf& conf, RngStream& rng) {  // noise.cpp:162-197
    return mc_trajectories(c, conf, rng, 1)[0];
}

// ------------------------------------------------------------------ variational
void AnsatzSpec::validate() const {  // variational.cpp:11-16
    require(n_params >= 0, "AnsatzSpec: negative parameter count");
    require(static_cast<bool>(builder), "AnsatzSpec: missing builder");
    require(shift_eligible.size() == static_cast<std::size_t>(n_params),
            "AnsatzSpec: eligibility tags do not match parameter count");
}

AnsatzSpec tfim_chain_ansatz(int n, int layers) {  // variational.cpp:18-36
    require(n >= 2, "tfim_chain_ansatz: n must be >= 2");
    require(layers >= 1, "tfim_chain_ansatz: layers must be >= 1");
    AnsatzSpec a;
    a.n_params = layers * (2 * n - 1);
    a.shift_eligible.assign(a.n_params, true);
    a.builder = [n, layers](const RealVector& theta) {
        Circuit c(n);
        for (int q = 0; q < n; ++q) c.h(q);
        int k = 0;
        for (int l = 0; l < layers; ++l) {
            for (int i = 0; i < n; ++i) c.rx(i, theta[k++]);
            for (int i = 0; i + 1 < n; ++i) c.rzz(i, i + 1, theta[k++]);
        }
        return c;
    };
    return a;
}

AnsatzSpec hea_ansatz(int n, int layers) {
    require(n >= 2 && layers >= 1, "hea_ansatz: n >= 2 and layers >= 1");
    AnsatzSpec a;
    a.n_params = 2 * n * layers;
    a.shift_eligible.assign(a.n_params, true);
    a.builder = [n, layers](const RealVector& theta) {
        Circuit c(n);
        int k = 0;
        for (int l = 0; l < layers; ++l) {
            for (int q = 0; q < n; ++q) c.ry(q, theta[k++]);
            for (int q = 0; q < n; ++q) c.rz(q, theta[k++]);
            for (int q = 0; q + 1 < n; ++q) c.cx(q, q + 1);
        }
        return c;
    };
    return a;
}

namespace {

template <class D>
bool same_matrix(const D& x, const D& y) {
    if (x.rows() != y.rows() || x.cols() != y.cols()) return false;
    for (std::int64_t i = 0; i < x.size(); ++i)
        if (x.data()[i] != y.data()[i]) return false;
    return true;
}

bool same_init(const std::optional<ComplexVector>& x, const std::optional<ComplexVector>& y) {
    if (x.has_value() != y.has_value()) return false;
    return !x || same_matrix(*x, *y);
}

std::uint64_t template_key(const Template& t, int n_params) {
    Fnv f;
    f.add(t.n);
    f.add(n_params);
    for (const qf_op& q : t.ops) {
        f.add(q.kind); f.add(q.q0); f.add(q.q1); f.add(q.slot); f.add(q.coef); f.add(q.offset); f.add(q.mat);
    }
    f.add(t.mats.data(), t.mats.size() * sizeof(double));
    f.add(t.init.has_value());
    if (t.init) f.add(t.init->data(), (size_t)t.init->size() * sizeof(cplx));
    return f.h;
}

// The builder cannot be mapped to one fixed template: energies then take the
// per-parameter-set path (per_theta_energies), the adjoint gradient rethrows.
struct TemplateUnavailable : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
void require_template(bool cond, const char* msg) {
    if (!cond) throw TemplateUnavailable(msg);
}

// Parameter-slot discovery: probe the opaque builder.  The
// builder is probed on every call and the compiled program is reused only
// while the discovered template (ops, slots, matrices, initial state) and
// n_params are unchanged: `builder` and `n_params` are public fields.
std::shared_ptr<ProgramHandle> ansatz_program(const AnsatzSpec& a) {
    struct Cache {
        std::map<std::pair<int, std::uint64_t>, std::shared_ptr<ProgramHandle>> progs;  // (precision, template key)
    };
    auto cache = std::static_pointer_cast<Cache>(a.device_cache);
    a.validate();
    const int P = a.n_params;
    RealVector t0 = RealVector::Zero(P), ta(P), tb(P), tc(P);
    for (int j = 0; j < P; ++j) {
        ta[j] = 1.0 + 1e-3 * j + 0.137;
        tb[j] = ta[j] * (2.0 + 1e-3 * j);
        tc[j] = std::cos(3.7 * j + 0.3) * 2.1 + 0.05;
    }
    const Circuit c0 = a.builder(t0), ca = a.builder(ta), cb = a.builder(tb), cc = a.builder(tc);
    for (const Circuit* c : {&ca, &cb, &cc}) {
        bool same = c->n == c0.n && c->ops.size() == c0.ops.size();
        for (size_t i = 0; same && i < c0.ops.size(); ++i)
            same = c->ops[i].name == c0.ops[i].name && c->ops[i].wires == c0.ops[i].wires;
        require_template(same, "AnsatzSpec: builder structure depends on theta (device path needs a fixed structure)");
        require_template(same_init(c->initial_state, c0.initial_state),
                "AnsatzSpec: theta feeds the initial state (not supported on the device path)");
    }
    std::vector<SlotMap> slots(c0.ops.size());
    for (size_t i = 0; i < c0.ops.size(); ++i) {
        const GateInstruction& op = c0.ops[i];
        if (!is_rotation(op.name)) {
            for (const Circuit* c : {&ca, &cb, &cc})
                require_template(c->ops[i].params == op.params && same_matrix(c->ops[i].matrix, op.matrix),
                        "AnsatzSpec: theta feeds a gate without a Pauli generator "
                        "(su4/unitary parameters are not supported on the device path)");
            continue;
        }
        const double o = op.params.at(0);
        const double da = ca.ops[i].params.at(0) - o, db = cb.ops[i].params.at(0) - o;
        if (da == 0.0 && db == 0.0) {
            require_template(cc.ops[i].params.at(0) == o, "AnsatzSpec: builder is not affine in theta");
            continue;
        }
        require_template(da != 0.0 && P > 0, "AnsatzSpec: builder is not affine in theta");
        int s = 0;
        double best = INFINITY;
        for (int j = 0; j < P; ++j) {
            const double d = std::abs(tb[j] / ta[j] - db / da);
            if (d < best) {
                best = d;
                s = j;
            }
        }
        const double coef = da / ta[s];
        const double pred = coef * tc[s] + o;
        require_template(std::abs(pred - cc.ops[i].params.at(0)) <= 1e-9 * std::max(1.0, std::abs(pred)),
                "AnsatzSpec: builder is not affine in a single theta slot");
        slots[i] = {s, coef, o};
    }
    const Template t = circuit_template(c0, &slots);
    const auto key = std::make_pair((int)g_prec, template_key(t, P));
    if (cache) {
        auto f = cache->progs.find(key);
        if (f != cache->progs.end()) return f->second;
    }
    auto prog = make_program(t, P);
    if (!cache) {
        cache = std::make_shared<Cache>();
        a.device_cache = cache;
    }
    if (cache->progs.size() >= 8) cache->progs.clear();  // bound the programs kept per spec
    cache->progs[key] = prog;
    return prog;
}

// The reference's own energy path (variational.cpp:38-52: build, run,
// expectation) for builders without a fixed template, one parameter set at a
// time, on the device: each circuit is a constant program whose generated
// kernels do not depend on angle values (they come from the kernel cache).
void per_theta_energies(const AnsatzSpec& a, const std::vector<double>& flat, int batch, const PauliSum* h,
                        const SparseCOO* hs, std::vector<double>& E) {
    const int P = a.n_params;
    E.assign(batch, 0.0);
    for (int b = 0; b < batch; ++b) {
        RealVector th(P);
        for (int j = 0; j < P; ++j) th[j] = flat[(size_t)b * P + j];
        const Circuit c = a.builder(th);
        auto prog = make_program(circuit_template(c, nullptr), 0);
        const double none = 0.0;
        if (h) {
            require(h->n == c.n, "expectation_pauli: size mismatch");
            check(qf_energy_grad_batch(ctx(), prog->p, observable(*h), 1, &none, &E[b], nullptr));
        } else {
            check(qf_sparse_energy(ctx(), prog->p, 1, &none, hs->dim, (std::int64_t)hs->nnz(), hs->rows.data(),
                                   hs->cols.data(), reinterpret_cast<const double*>(hs->vals.data()), 0, &E[b]));
        }
    }
}

void batch_eval(const AnsatzSpec& a, const std::vector<double>& flat, int batch, const PauliSum& h,
                std::vector<double>& E, std::vector<double>* G) {
    std::shared_ptr<ProgramHandle> prog;
    try {
        prog = ansatz_program(a);
    } catch (const TemplateUnavailable&) {
        if (G) throw;  // the adjoint gradient needs the template
        per_theta_energies(a, flat, batch, &h, nullptr, E);
        return;
    }
    E.assign(batch, 0.0);
    if (G) G->assign((size_t)batch * a.n_params, 0.0);
    if (batch == 0) return;
    check(qf_energy_grad_batch(ctx(), prog->p, observable(h), batch, flat.data(), E.data(), G ? G->data() : nullptr));
}

}  // namespace

double energy(const AnsatzSpec& ansatz, const RealVector& theta, const PauliSum& h) {  // variational.cpp:38-43
    ansatz.validate();
    require(theta.size() == ansatz.n_params, "energy: parameter count mismatch");
    std::vector<double> flat(theta.data(), theta.data() + theta.size()), E;
    batch_eval(ansatz, flat, 1, h, E, nullptr);
    return E[0];
}

double energy(const AnsatzSpec& ansatz, const RealVector& theta, const SparseCOO& h) {  // variational.cpp:45-52
    ansatz.validate();
    require(theta.size() == ansatz.n_params, "energy: parameter count mismatch");
    std::shared_ptr<ProgramHandle> prog;
    try {
        prog = ansatz_program(ansatz);
    } catch (const TemplateUnavailable&) {
        std::vector<double> flat(theta.data(), theta.data() + theta.size()), Es;
        per_theta_energies(ansatz, flat, 1, nullptr, &h, Es);
        return Es[0];
    }
    double E = 0.0;
    check(qf_sparse_energy(ctx(), prog->p, 1, theta.data(), h.dim, (std::int64_t)h.nnz(), h.rows.data(),
                           h.cols.data(), reinterpret_cast<const double*>(h.vals.data()), 0, &E));
    return E;
}

RealVector gradient(const AnsatzSpec& ansatz, const RealVector& theta, const PauliSum& h, GradMode mode,
                    double fd_step, int /*workers: results never depend on it*/) {  // variational.cpp:54-81
    ansatz.validate();
    require(theta.size() == ansatz.n_params, "gradient: parameter count mismatch");
    const int P = ansatz.n_params;
    RealVector grad(P);
    if (mode == GradMode::adjoint) {
        std::vector<double> flat(theta.data(), theta.data() + P), E, G;
        batch_eval(ansatz, flat, 1, h, E, &G);
        for (int j = 0; j < P; ++j) grad[j] = G[j];
        return grad;
    }
    if (mode == GradMode::parameter_shift) {
        for (int j = 0; j < P; ++j)
            require(ansatz.shift_eligible[j], "gradient: parameter not shift-eligible, use finite_diff");
    } else {
        require(fd_step > 0.0, "gradient: finite-diff step must be positive");
    }
    const double shift = mode == GradMode::parameter_shift ? M_PI / 2.0 : fd_step;
    const double denom = mode == GradMode::parameter_shift ? 2.0 : 2.0 * fd_step;
    std::vector<double> flat((size_t)2 * P * P), E;  // all 2P shifted energies in one device batch
    for (int j = 0; j < P; ++j)
        for (int s = 0; s < 2; ++s) {
            double* row = flat.data() + ((size_t)2 * j + s) * P;
            for (int i = 0; i < P; ++i) row[i] = theta[i];
            row[j] = theta[j] + (s == 0 ? shift : -shift);
        }
    batch_eval(ansatz, flat, 2 * P, h, E, nullptr);
    for (int j = 0; j < P; ++j) grad[j] = (E[2 * j] - E[2 * j + 1]) / denom;
    return grad;
}

void energy_gradient_batch(const AnsatzSpec& ansatz, const std::vector<RealVector>& thetas, const PauliSum& h,
                           std::vector<double>& energies, std::vector<RealVector>* grads) {
    ansatz.validate();
    const int P = ansatz.n_params, B = (int)thetas.size();
    std::vector<double> flat((size_t)B * P), G;
    for (int b = 0; b < B; ++b) {
        require(thetas[b].size() == P, "energy: parameter count mismatch");
        std::memcpy(flat.data() + (size_t)b * P, thetas[b].data(), sizeof(double) * P);
    }
    batch_eval(ansatz, flat, B, h, energies, grads ? &G : nullptr);
    if (grads) {
        grads->assign(B, RealVector(P));
        for (int b = 0; b < B; ++b)
            for (int j = 0; j < P; ++j) (*grads)[b][j] = G[(size_t)b * P + j];
    }
}

void adam_step(AdamState& state, RealVector& theta, const RealVector& grad, double lr, double beta1, double beta2,
               double eps) {  // variational.cpp:83-101
    require(theta.size() == grad.size(), "adam_step: shape mismatch");
    if (state.t == 0) {
        state.m = RealVector::Zero(theta.size());
        state.v = RealVector::Zero(theta.size());
    }
    require(state.m.size() == theta.size(), "adam_step: state shape mismatch");
    ++state.t;
    state.m = beta1 * state.m + (1.0 - beta1) * grad;
    state.v = beta2 * state.v + (1.0 - beta2) * grad.cwiseProduct(grad);
    const double c1 = 1.0 - std::pow(beta1, state.t);
    const double c2 = 1.0 - std::pow(beta2, state.t);
    for (std::int64_t i = 0; i < theta.size(); ++i) {
        const double mhat = state.m[i] / c1;
        const double vhat = state.v[i] / c2;
        theta[i] -= lr * mhat / (std::sqrt(vhat) + eps);
    }
}

VqeResult vqe_run(const AnsatzSpec& ansatz, const std::vector<RealVector>& theta0_batch, const PauliSum& h, int steps,
                  double lr, GradMode grad_mode, int /*workers: results never depend on it*/) {  // variational.cpp:103-143
    ansatz.validate();
    require(!theta0_batch.empty(), "vqe_run: empty batch");
    require(steps >= 1, "vqe_run: steps must be >= 1");
    const int B = (int)theta0_batch.size(), P = ansatz.n_params;
    if (grad_mode == GradMode::parameter_shift)
        for (int j = 0; j < P; ++j)
            require(ansatz.shift_eligible[j], "gradient: parameter not shift-eligible, use finite_diff");
    std::vector<double> flat((size_t)B * P);
    for (int b = 0; b < B; ++b) {
        require(theta0_batch[b].size() == P, "gradient: parameter count mismatch");
        std::memcpy(flat.data() + (size_t)b * P, theta0_batch[b].data(), sizeof(double) * P);
    }
    std::shared_ptr<ProgramHandle> prog;
    try {
        prog = ansatz_program(ansatz);
    } catch (const TemplateUnavailable&) {
        if (grad_mode == GradMode::adjoint) throw;
        // no fixed template: the reference's loop (variational.cpp:118-141) over
        // the per-parameter-set energy path
        VqeResult out;
        out.traces.assign(B, {});
        out.final_thetas.assign(B, RealVector(P));
        for (int b = 0; b < B; ++b) {
            RealVector theta = theta0_batch[b];
            AdamState adam;
            for (int st = 0; st < steps; ++st) {
                out.traces[b].push_back(energy(ansatz, theta, h));
                adam_step(adam, theta, gradient(ansatz, theta, h, grad_mode, 1e-5, 1), lr);
            }
            out.final_thetas[b] = theta;
        }
        out.best_energy = INFINITY;
        for (int b = 0; b < B; ++b) {
            const double e = energy(ansatz, out.final_thetas[b], h);
            out.traces[b].push_back(e);
            if (e < out.best_energy) {
                out.best_energy = e;
                out.best_index = b;
            }
        }
        return out;
    }
    // theta, the Adam moments and the traces stay on the device for all steps
    // (one native call; the batch advances in lock step, one host copy at the end)
    std::vector<double> tr((size_t)B * (steps + 1)), fin((size_t)B * P);
    const int mode = grad_mode == GradMode::adjoint ? QF_GRAD_ADJOINT
                     : grad_mode == GradMode::finite_diff ? QF_GRAD_FINITE_DIFF : QF_GRAD_PARAMETER_SHIFT;
    VqeResult out;
    check(qf_vqe_run(ctx(), prog->p, observable(h), B, flat.data(), steps, lr, mode, 1e-5, tr.data(), fin.data(),
                     &out.best_energy, &out.best_index));
    out.traces.assign(B, {});
    out.final_thetas.assign(B, RealVector(P));
    for (int b = 0; b < B; ++b) {
        out.traces[b].assign(tr.begin() + (size_t)b * (steps + 1), tr.begin() + (size_t)(b + 1) * (steps + 1));
        for (int j = 0; j < P; ++j) out.final_thetas[b][j] = fin[(size_t)b * P + j];
    }
    return out;
}

}  // namespace qforge
