// TEST INFRASTRUCTURE ONLY: compiled against the reference's own, Eigen-free
// proj/include/qforge/rng.hpp (include path set by oracle/Makefile; the header
// is not copied into this repo).  Prints RNG known answers and the draw order of
// tests/helpers.hpp:52-63 random_pauli_sum (including the complex-weight case,
// whose argument-evaluation order is compiler-defined) so the C oracle's
// restatement can be pinned to the real thing.  Output goes to oracle/_ref/.
#include <complex>
#include <cstdio>
#include <vector>

#include "qforge/rng.hpp"

int main() {
    using qforge::RngStream;
    {
        RngStream r(3);
        for (int i = 0; i < 8; ++i) std::printf("normal3 %.17g\n", r.normal());
    }
    {
        RngStream r(7);
        for (int i = 0; i < 4; ++i) std::printf("u64_7 %llu\n", (unsigned long long)r.next_u64());
    }
    {
        RngStream r(0);
        auto kids = r.split(8);
        for (int i = 0; i < 8; ++i) std::printf("split0 %d %.17g\n", i, kids[i].normal());
    }
    {
        RngStream r(11);
        for (int i = 0; i < 16; ++i) std::printf("below5 %llu\n", (unsigned long long)r.uniform_below(5));
        for (int i = 0; i < 4; ++i) std::printf("uniform %.17g\n", r.uniform());
    }
    {
        // helpers.hpp:52-63 with real_weights = false
        RngStream r(13);
        for (int t = 0; t < 4; ++t) {
            std::printf("rps_codes");
            for (int q = 0; q < 5; ++q) std::printf(" %d", (int)r.uniform_below(4));
            std::complex<double> w = std::complex<double>(r.normal(), r.normal());
            std::printf("\nrps_w %.17g %.17g\n", w.real(), w.imag());
        }
    }
    return 0;
}
