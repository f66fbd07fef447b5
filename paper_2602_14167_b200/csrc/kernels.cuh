// kernels.cuh -- launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "plan.h"

namespace qfb {

struct SweepArgs {
    void* psi;                 // [B][N] complex (float2 / double2)
    void* lam;                 // adjoint state (backward only)
    const double* theta;       // [B_total][P]
    int P;
    int n;
    int batch_offset;          // global index of blockIdx.y == 0 (theta rows)
    int from_zero;             // forward sweep 0 builds |0..0> in-tile
    DevSweep sw;               // this sweep (by value)
    const DevPhase* phases;
    const DevOp* ops;
    const DevGate* gates;
    const double* cmats;       // constant matrices [n][16][2]
    double* tap_part;          // [B][n_taps_total][tiles]
    int n_taps_total;
};

struct HArgs {
    const void* psi;
    void* lam;
    int n, kh;
    const DevGroup* groups;
    int n_groups;
    const DevTerm* terms;
    int write_lam;
    int use_imag;
    double* epart;             // [B][tiles]
};

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
cudaError_t launch_init_state(int prec, void* psi, const void* init, int n, int batch,
                              cudaStream_t s);
cudaError_t launch_reduce(const ReduceArgs& a, int batch, cudaStream_t s);
cudaError_t launch_gather_grads(const double* tapsum, int n_taps, const int* slot_ptr,
                                const int* slot_taps, const double* slot_coef, int P,
                                int batch, double* grads /* [B][P] */, cudaStream_t s);
cudaError_t launch_adam(int count, double* theta, double* m, double* v, const double* g,
                        double lr, double b1, double b2, double eps, double c1, double c2,
                        cudaStream_t s);
cudaError_t launch_convert_state(int prec, const void* src, double* dst, int64_t count,
                                 cudaStream_t s);

}  // namespace qfb
