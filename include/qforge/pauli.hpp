// qforge/pauli.hpp -- Pauli-sum IR (reference include/qforge/pauli.hpp:13-41):
// PauliTerm, PauliSum::add / add_word, tfim_terms, heisenberg_terms, pauli_sum_to_coo.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include <string>

#include "qforge/common.hpp"
#include "qforge/lattice.hpp"
#include "qforge/sparse.hpp"

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

    // wire format {"n","terms":[{"codes","w_im","w_re"}]} (pauli.cpp:29-50)
    std::string to_json() const;
    static PauliSum from_json(const std::string& text);

    // device copy (qf_observable), rebuilt when the terms change (content-keyed)
    mutable std::shared_ptr<void> device_cache;
};

// canonical COO of the sum, built on the GPU (pauli.cpp:89-153); `workers` is
// accepted for signature compatibility (the output never depends on it)
SparseCOO pauli_sum_to_coo(const PauliSum& h, int n_guard = 26, std::size_t workers = 1);

PauliSum tfim_terms(const Lattice& l, double g);
PauliSum heisenberg_terms(const Lattice& l, double jx, double jy, double jz);

}  // namespace qforge
