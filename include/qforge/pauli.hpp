// qforge/pauli.hpp -- Pauli-sum IR (reference include/qforge/pauli.hpp:13-41):
// PauliTerm, PauliSum::add / add_word, tfim_terms, heisenberg_terms.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "qforge/common.hpp"
#include "qforge/lattice.hpp"

namespace qforge {

// Pauli codes: 0=I, 1=X, 2=Y, 3=Z.
struct PauliTerm {
    cplx weight;
    std::vector<int> codes;  // length n
};

struct PauliSum {
    int n = 0;
    std::vector<PauliTerm> terms;

    void add(cplx weight, const std::vector<int>& codes);
    void add_word(cplx weight, const std::vector<std::pair<int, int>>& site_codes);

    // device copy (qf_observable), rebuilt when the terms change
    mutable std::shared_ptr<void> device_cache;
    mutable std::size_t device_cache_terms = 0;
};

PauliSum tfim_terms(const Lattice& l, double g);
PauliSum heisenberg_terms(const Lattice& l, double jx, double jy, double jz);

}  // namespace qforge
