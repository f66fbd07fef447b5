// qforge/variational.hpp -- drop-in for the reference's
// include/qforge/variational.hpp:14-57 (AnsatzSpec, tfim_chain_ansatz, energy,
// GradMode, gradient, AdamState, adam_step, VqeResult, vqe_run).
// Additive: GradMode::adjoint, energy_gradient_batch, hea_ansatz.
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/common.hpp"
#include "qforge/pauli.hpp"
#include "qforge/rng.hpp"

namespace qforge {

struct AnsatzSpec {
    int n_params = 0;
    std::function<Circuit(const RealVector&)> builder;
    std::vector<bool> shift_eligible;

    void validate() const;

    // compiled device program (slot-affine template discovered by probing the builder)
    mutable std::shared_ptr<void> device_cache;
};

AnsatzSpec tfim_chain_ansatz(int n, int layers);
AnsatzSpec hea_ansatz(int n, int layers);  // synthetic HEA of the benchmark configs

double energy(const AnsatzSpec& ansatz, const RealVector& theta, const PauliSum& h);
double energy(const AnsatzSpec& ansatz, const RealVector& theta, const SparseCOO& h);  // COO operator path

enum class GradMode { parameter_shift, finite_diff, adjoint };

RealVector gradient(const AnsatzSpec& ansatz, const RealVector& theta, const PauliSum& h, GradMode mode,
                    double fd_step = 1e-5, int workers = 1);

// energies[b] and gradients[b] (adjoint) for a batch of parameter sets, one device pass
void energy_gradient_batch(const AnsatzSpec& ansatz, const std::vector<RealVector>& thetas, const PauliSum& h,
                           std::vector<double>& energies, std::vector<RealVector>* grads);

struct AdamState {
    RealVector m;
    RealVector v;
    int t = 0;
};

void adam_step(AdamState& state, RealVector& theta, const RealVector& grad, double lr, double beta1 = 0.9,
               double beta2 = 0.999, double eps = 1e-8);

struct VqeResult {
    std::vector<std::vector<double>> traces;
    std::vector<RealVector> final_thetas;
    double best_energy = 0.0;
    int best_index = -1;
};

VqeResult vqe_run(const AnsatzSpec& ansatz, const std::vector<RealVector>& theta0_batch, const PauliSum& h,
                  int steps, double lr, GradMode grad_mode, int workers = 1);

}  // namespace qforge
