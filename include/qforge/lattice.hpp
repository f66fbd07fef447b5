// qforge/lattice.hpp -- the geometry the hot path uses: build_lattice(chain)
// and its order-1 neighbour shell (reference src/lattice.cpp:29-48, 89-170).
// Other lattice kinds are out of scope and throw.
#pragma once

#include <map>
#include <utility>
#include <vector>

#include "qforge/common.hpp"

namespace qforge {

enum class LatticeKind { chain, square, triangular, honeycomb, kagome, custom };

struct Lattice {
    LatticeKind kind = LatticeKind::chain;
    double lattice_constant = 1.0;
    int n_sites = 0;
    std::map<int, std::vector<std::pair<int, int>>> edges_by_order;  // order -> (i < j)
    std::size_t num_sites() const { return (std::size_t)n_sites; }
};

Lattice build_lattice(LatticeKind kind, const std::vector<int>& size, const std::vector<bool>& pbc,
                      double lattice_constant = 1.0, int neighbor_order = 1);

}  // namespace qforge
