// kernels.cuh -- launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "plan.h"

namespace qfb {

struct ReduceArgs {
    const double* part;        // [B][count][tiles]
    int count, tiles;
    double* out;               // [B][count]
};

// returns dynamic smem bytes needed (for attribute setup / occupancy)
size_t sweep_smem_bytes(int prec, bool bwd, const DevSweep& sw, int max_mat, int max_taps);

cudaError_t launch_sweep(int prec, bool bwd, const SweepArgs& a, int batch, int max_mat,
                         int max_taps, cudaStream_t s);
cudaError_t launch_hpsi(int prec, const HArgs& a, int batch, cudaStream_t s);
cudaError_t launch_mats(int prec, bool adj, const DevOp* ops, const int* goff, int n_ops, const DevGate* gates,
                        const double* cmats, const double* theta, int P, int batch_offset, void* out, int stride,
                        int pass_base, int batch, cudaStream_t s,
                        size_t cmats_stride = 0);
cudaError_t launch_init_state(int prec, void* psi, const void* init, int n, int batch,
                              cudaStream_t s);
cudaError_t launch_reduce(const ReduceArgs& a, int batch, cudaStream_t s);
cudaError_t launch_gather_grads(const double* tapsum, int n_taps, const int* slot_ptr,
                                const int* slot_taps, const double* slot_coef, int P,
                                int batch, double* grads /* [B][P] */, cudaStream_t s);
cudaError_t launch_shift_thetas(int B, int P, const double* theta, double shift, double* out, cudaStream_t s);
cudaError_t launch_shift_grad(int B, int P, const double* E, double denom, double* g, cudaStream_t s);
cudaError_t launch_adam(int count, double* theta, double* m, double* v, const double* g,
                        double lr, double b1, double b2, double eps, double c1, double c2,
                        cudaStream_t s);
cudaError_t launch_convert_state(int prec, const void* src, double* dst, int64_t count,
                                 cudaStream_t s);

}  // namespace qfb

namespace qfb {

// ---- pauli_sum_to_coo (reference src/pauli.cpp:89-153) ----
struct CooGroup {          // terms sharing one flip mask
    uint64_t flip;
    int32_t term_begin, term_end;
};
struct CooTerm {
    uint64_t z;
    double c_re, c_im;     // w * i^y
};
// Column ranking for <= 32 flip groups.  Binary trie over the ascending flip
// masks: an internal node at bit d splits the group range [lo, hi) at mid (first
// flip with bit d set), and rows with bit d set list [mid, hi) before [lo, mid).
// As a difference array over the group index each such node contributes
// +cnt[mid,hi) at lo, -cnt[lo,hi) at mid and +cnt[lo,mid) at hi; one event per
// contribution, sorted by position (cnt = non-zero groups under `mask`).
struct CooEvent {
    int32_t pos, d, sign;
    uint32_t mask;
};
// nnz per row (values summed per flip group, exact zeros dropped)
cudaError_t launch_coo_count(const CooGroup* g, int n_groups, const CooTerm* t, int n_terms, int n, int64_t* counts,
                             cudaStream_t s);
// exclusive scan counts -> offsets (offsets[dim] = nnz); scratch via cub
cudaError_t coo_scan(const int64_t* counts, int64_t* offsets, int64_t dim, void* scratch, size_t* scratch_bytes,
                     cudaStream_t s);
// E partials of <psi|H|psi> for a COO H (sparse.cpp:44-51 + variational.cpp:45-52):
// block j sums Re(conj(psi[r_k]) v_k psi[c_k]) over its contiguous nnz range,
// fixed order; launch_reduce(count 1, tiles = blocks) finishes.  Returns blocks.
int coo_energy_blocks(int64_t nnz);
cudaError_t launch_coo_energy(int prec, const int64_t* rows, const int64_t* cols, const double2* vals, int64_t nnz,
                              const void* psi, double* part, cudaStream_t s);
// ---- trajectories (reference experiments.cpp:210-250, circuit.cpp:391-429) ----
// Up to kMeasMax projective measurements per state and round: hist[b][beta] =
// sum |psi|^2 over amplitudes whose measured bits equal beta (fixed order);
// mipt_decide replays measure_collapse sequentially on the histogram; project
// zeroes the rejected amplitudes and rescales the rest.
constexpr int kMeasMax = 8;
struct MeasRound {
    int count;                   // measurements of this state in this round
    int pos[kMeasMax];           // memory bit positions (n - 1 - wire), in order
    double u[kMeasMax];          // the uniform drawn by measure_collapse
};
cudaError_t launch_meas_hist(int prec, const void* psi, int n, int batch, const MeasRound* rounds, int max_count,
                             double* hist, cudaStream_t s);
cudaError_t launch_meas_decide(const MeasRound* rounds, const double* hist, int batch, uint32_t* mask, uint32_t* bits,
                               double* scale, int* outcomes, cudaStream_t s);
cudaError_t launch_meas_project(int prec, void* psi, int n, int batch, const MeasRound* rounds, const uint32_t* mask,
                                const uint32_t* bits, const double* scale, cudaStream_t s);
// one inverse-CDF sample per state (u[b] in [0, 1)); csum: [batch][2^(n - sample_chunk_bits(n))]
int sample_chunk_bits(int n);
cudaError_t launch_sample(int prec, const void* psi, int n, int batch, const double* u, double* csum, int64_t* hit,
                          cudaStream_t s);
// one 1- or 2-qubit operator (memory bit positions p0 = wires[0], p1 = wires[1] or -1)
// on every state; m = [D][D] complex row-major, shared or one per state
cudaError_t launch_apply_local(int prec, void* psi, int n, int batch, int p0, int p1, const double2* m, bool per_state,
                               cudaStream_t s);
// k-wire operator on one complex128 state (apply_local_unitary): d_pos[k] = memory
// bit positions (wires[0] first = most significant local bit), d_u = U row-major
// (k <= 4), d_ut = U column-major (k >= 5, k <= 13)
cudaError_t launch_apply_unitary(double2* psi, int n, int k, const int* d_pos, const double2* d_u, const double2* d_ut,
                                 cudaStream_t s);
// number of fixed-order rho partials per state of launch_apply_rho
int local_rho_parts(int n);
cudaError_t launch_set_basis0(int prec, void* psi, int n, int batch, cudaStream_t s);
// noise step: operator m on wires (p0[, p1]) then the local rho partials of the
// result on those wires ([batch][local_rho_parts(n)][D][D], fixed order)
cudaError_t launch_apply_rho(int prec, void* psi, int n, int batch, int p0, int p1, const double2* m, bool per_state,
                             double2* rho, cudaStream_t s);
// the same with a pending per-trajectory operator kp ([batch][DP][DP]) on the
// disjoint wires (q0[, q1]) applied first, in the same pass
cudaError_t launch_apply2_rho(int prec, void* psi, int n, int batch, int q0, int q1, const double2* kp, int p0,
                              int p1, const double2* g, double2* rho, cudaStream_t s);
// per-trajectory Kraus branch pick for one channel application (kraus: [k][4][4]
// complex, channel = k0 .. k1-1; u[b * u_stride + app]); kout [batch][D][D],
// logp[b] += log p_pick; err = 1 if all branch probabilities vanish
cudaError_t launch_kraus_pick(const double2* rho, int parts, int D, const double* kraus, int k0, int k1, const double* u,
                              int u_stride, int app, double2* kout, double* logp, int* err, int batch, cudaStream_t s);

// eigenvalues (ascending) of `batch` Hermitian m x m matrices (column-major, both
// triangles, overwritten): Householder tridiagonalisation + Sturm bisection (eig.cu);
// d, e: [batch][m] scratch each, w: [batch][m]; m <= 2048
cudaError_t launch_hermitian_eigvals(double2* A, int m, int batch, double* d, double* e, double* w, cudaStream_t s);

// rows / cols ascending per row, complex128 values
cudaError_t launch_coo_write(const CooGroup* g, int n_groups, const CooTerm* t, int n_terms, const CooEvent* ev,
                             int n_ev, int n, const int64_t* offsets,
                             int64_t* rows, int64_t* cols, double2* vals, cudaStream_t s);

}  // namespace qfb
