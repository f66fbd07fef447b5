// test_json.cpp -- the reference's JSON wire-format tests
// (proj/tests/test_circuit.cpp:323-328 "circuit json round trip",
//  proj/tests/test_hamiltonian.cpp:249-260 "pauli sum json round trip")
// on the drop-in headers, plus malformed-input errors.  No device needed.
// Usage: test_json            -> runs the checks, prints "ok N"
//        test_json dump       -> prints the fixed documents (compared with the
//                                Python mirror by tests/test_cpp_json.py)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <stdexcept>
#include <type_traits>

#include "qforge/circuit.hpp"
#include "qforge/pauli.hpp"
#include "qforge/rng.hpp"

using namespace qforge;

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                     \
    do {                                                             \
        ++g_checks;                                                  \
        if (!(c)) {                                                  \
            ++g_fail;                                                \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
        }                                                            \
    } while (0)

static Circuit fixed_circuit() {
    Circuit c(3);
    c.h(0).rx(1, 0.25).ry(2, -1.5e-7).rz(0, 3.0).rzz(0, 2, 1e20).cx(1, 2).cz(0, 1).su4(0, 1, {0.1, 0.2, 0.3, 0.4, 0.5,
                                                                                                0.6, 0.7, 0.8, 0.9, 1.0,
                                                                                                1.1, 1.2, 1.3, 1.4, 1.5});
    ComplexMatrix u(2, 2);
    const double s = std::sqrt(0.5);
    u(0, 0) = cplx(s, 0);
    u(0, 1) = cplx(0, s);
    u(1, 0) = cplx(0, s);
    u(1, 1) = cplx(s, 0);
    c.unitary({2}, u);
    return c;
}

static PauliSum fixed_sum() {
    PauliSum h;
    h.n = 3;
    h.add(cplx(1.0, 0.0), {1, 0, 3});
    h.add(cplx(-0.5, 0.125), {2, 2, 0});
    h.add(cplx(1e-5, -3.0), {0, 0, 0});
    return h;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "dump") == 0) {
        std::cout << fixed_circuit().to_json() << "\n" << fixed_sum().to_json() << "\n";
        return 0;
    }
    {  // Eigen-compatible shim: column-major data(), row-order comma init, real cwiseAbs,
       // distinct matrix / vector types, matrix * vector -> vector
        ComplexMatrix m(2, 3);
        m << cplx(1, 0), cplx(2, 0), cplx(3, 0), cplx(4, 0), cplx(5, 0), cplx(6, 1);
        CHECK(m(0, 1) == cplx(2, 0) && m(1, 0) == cplx(4, 0) && m(1, 2) == cplx(6, 1));
        CHECK(m.data()[0] == cplx(1, 0) && m.data()[1] == cplx(4, 0) && m.data()[2] == cplx(2, 0));  // columns
        const double mx = m.cwiseAbs().maxCoeff();
        CHECK(std::abs(mx - std::abs(cplx(6, 1))) < 1e-15);
        ComplexVector v = ComplexVector::Zero(3);
        v[0] = 1.0;
        v[2] = cplx(0, 1);
        const ComplexVector mv = m * v;
        CHECK(mv.size() == 2 && mv[0] == cplx(1, 3) && mv[1] == cplx(4, 0) + cplx(6, 1) * cplx(0, 1));
        static_assert(!std::is_same_v<ComplexMatrix, ComplexVector>, "distinct types, as in Eigen");
        const ComplexMatrix a = m.adjoint();
        CHECK(a.rows() == 3 && a.cols() == 2 && a(2, 1) == cplx(6, -1));
    }
    {  // round trips preserve every field exactly
        Circuit c = fixed_circuit();
        Circuit b = Circuit::from_json(c.to_json());
        CHECK(b.n == c.n && b.d == c.d && b.ops.size() == c.ops.size());
        for (size_t i = 0; i < c.ops.size() && i < b.ops.size(); ++i) {
            CHECK(b.ops[i].name == c.ops[i].name);
            CHECK(b.ops[i].wires == c.ops[i].wires);
            CHECK(b.ops[i].params == c.ops[i].params);
            if (c.ops[i].name == Gate::unitary)
                for (std::int64_t k = 0; k < c.ops[i].matrix.size(); ++k)
                    CHECK(b.ops[i].matrix.data()[k] == c.ops[i].matrix.data()[k]);
        }
        CHECK(b.to_json() == c.to_json());
    }
    {  // pauli sum json round trip (test_hamiltonian.cpp:249-260), random complex weights
        RngStream rng(2);
        PauliSum h;
        h.n = 3;
        for (int t = 0; t < 4; ++t) {
            std::vector<int> codes;
            for (int q = 0; q < 3; ++q) codes.push_back((int)rng.uniform_below(4));
            const double im = rng.normal(), re = rng.normal();
            h.add(cplx(re, im), codes);
        }
        PauliSum back = PauliSum::from_json(h.to_json());
        CHECK(back.n == h.n && back.terms.size() == h.terms.size());
        for (size_t i = 0; i < h.terms.size() && i < back.terms.size(); ++i) {
            CHECK(back.terms[i].codes == h.terms[i].codes);
            CHECK(back.terms[i].weight == h.terms[i].weight);  // shortest round-trip doubles: exact
        }
    }
    {  // malformed input and unknown names raise invalid_argument (nlohmann parse_error / gate_from_name)
        auto throws = [](auto f) {
            try {
                f();
            } catch (const std::invalid_argument&) {
                return true;
            } catch (...) {
                return false;
            }
            return false;
        };
        CHECK(throws([] { Circuit::from_json("{\"n\":2,\"ops\":[{\"name\":\"foo\",\"wires\":[0],\"params\":[]}]}"); }));
        CHECK(throws([] { Circuit::from_json("{\"n\":2,\"ops\":[}"); }));
        CHECK(throws([] { Circuit::from_json("{\"ops\":[]}"); }));
        CHECK(throws([] { PauliSum::from_json("{\"n\":2,\"terms\":[{\"w_re\":1.0,\"codes\":[1,0]}]}"); }));
        CHECK(throws([] { PauliSum::from_json("{\"n\":2,\"terms\":[{\"w_re\":1.0,\"w_im\":0,\"codes\":[1,7]}]}"); }));
        CHECK(throws([] { Circuit::from_json("{\"n\":2,\"ops\":[{\"name\":\"h\",\"wires\":[5],\"params\":[]}]}"); }));
    }
    std::printf("%s %d checks, %d failed\n", g_fail ? "FAIL" : "ok", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
