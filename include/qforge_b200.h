/*
 * qforge_b200.h -- C-ABI of the B200 batched state-vector VQE engine.
 *
 * Plain C: pointers, sizes, int status codes; no C++/torch types.  Every entry
 * point replaces one piece of the reference qforge hot path (paths relative to
 * /root/reference/proj):
 *
 *   qf_program_create     <- Circuit / GateInstruction / Circuit::gate validation
 *                            (include/qforge/circuit.hpp:14-83, src/circuit.cpp:178-200)
 *                            + gate_matrix (src/circuit.cpp:202-302), compiled once
 *                            into fused tile sweeps instead of rebuilt per energy call
 *   qf_observable_create  <- PauliSum::add / compile_term (include/qforge/pauli.hpp:13-30,
 *                            src/pauli.cpp:12-27, 54-85)
 *   qf_run_state          <- run(const Circuit&, guard) (src/circuit.cpp:304-317)
 *   qf_expectation        <- expectation_pauli(psi, obs) (src/circuit.cpp:319-347)
 *   qf_energy_grad_batch  <- energy() + gradient() for a batch of parameter sets
 *                            (src/variational.cpp:38-81, batch loop of vqe_run :114-131);
 *                            gradient by the adjoint method (GradMode::adjoint, new)
 *   qf_adam_step_device   <- adam_step (src/variational.cpp:83-101) on device-resident
 *                            theta/m/v for vqe_run (src/variational.cpp:103-143)
 *   qf_ctx_set_comm       <- parallel_for (include/qforge/parallel.hpp:11-26): batch or
 *                            term sharding across GPUs, one NCCL all-reduce per call
 *
 * Conventions kept from the reference:
 *   - site 0 is the most significant bit of a basis index (circuit.cpp:87, :329);
 *   - states are complex amplitudes, interleaved (re, im), like std::complex<double>;
 *   - precondition failures return QF_EINVAL (the C++ shim maps it to
 *     std::invalid_argument, common.hpp:24-26); everything else is a runtime
 *     failure (std::runtime_error).  qf_last_error() has the message.
 *   - batch-sharded results never depend on the number of GPUs (parallel.hpp:9-10):
 *     every batch slot has exactly one owner and the all-reduce adds exact zeros.
 *     Term-sharded results (one large state, QF_SHARD_TERMS) equal the 1-GPU
 *     result up to floating-point summation order (each rank sums its own term
 *     block; measured <= 1e-12 relative, tests/test_gpu_api.py virtual ranks).
 *
 * Calls are synchronous (they return after results are on the host) except the
 * *_device variants, which are stream-ordered on the context's stream.
 * A context is not thread-safe; one context per GPU per process.
 */
#ifndef QFORGE_B200_H
#define QFORGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QF_ABI_VERSION 1

enum qf_status {
    QF_OK = 0,
    QF_EINVAL = 1,   /* precondition violated (reference: require() -> invalid_argument) */
    QF_ERUNTIME = 2, /* runtime failure (reference: runtime_error) */
    QF_ENOMEM = 3,
    QF_ECUDA = 4,
    QF_ENCCL = 5
};

enum qf_precision { QF_C64 = 0, QF_C128 = 1 };

/* Gate kinds: same numbering as qforge::Gate (include/qforge/circuit.hpp:14-23). */
enum qf_gate {
    QF_H = 0, QF_X, QF_Y, QF_Z, QF_S,
    QF_RX, QF_RY, QF_RZ, QF_RZZ,
    QF_CX, QF_CZ,
    QF_SU4, QF_CSUM, QF_SUBSPACE_RY, QF_SUBSPACE_RZ,
    QF_UNITARY
};

/* One gate of a parameterised circuit template.  The rotation angle is
 *   param = coef * theta[slot] + offset   (slot >= 0)
 *   param = offset                        (slot <  0)
 * This is GateInstruction{name, wires, params} (circuit.hpp:27-32) with the
 * theta -> params map of AnsatzSpec::builder (variational.hpp:14-21) made
 * explicit.  q1 = -1 for one-qubit gates.  QF_SU4 / QF_UNITARY take a constant
 * matrix: mat indexes the `mats` table of qf_program_create (row-major 4x4
 * complex128, a one-qubit matrix in its top-left 2x2 corner). */
typedef struct qf_op {
    int32_t kind;
    int32_t q0;
    int32_t q1;
    int32_t slot;
    double coef;
    double offset;
    int32_t mat;
    int32_t reserved;
} qf_op;

typedef struct qf_ctx qf_ctx;
typedef struct qf_program qf_program;
typedef struct qf_observable qf_observable;

/* Build / library info. */
int qf_abi_version(void);
const char* qf_last_error(void);

/* ---- context: one per GPU ---- */
int qf_ctx_create(int device, qf_ctx** out);
int qf_ctx_destroy(qf_ctx* ctx);
/* Memory budget (bytes) for batch state buffers; 0 = automatic (about 60% of free HBM). */
int qf_ctx_set_memory_budget(qf_ctx* ctx, size_t bytes);
/* Multi-GPU: one process per GPU.  Rank 0 calls qf_nccl_unique_id, ships the
 * 128 bytes to the other ranks (e.g. torch.distributed broadcast), then every
 * rank calls qf_ctx_set_comm.  world == 1 with an all-zero id detaches; world == 1
 * with a real id builds a single-rank communicator (exercises the collective
 * path on one GPU). */
int qf_nccl_unique_id(uint8_t out[128]);
int qf_ctx_set_comm(qf_ctx* ctx, int rank, int world, const uint8_t unique_id[128]);
/* Stream (cudaStream_t as void*) that *_device calls are ordered on. */
void* qf_ctx_stream(qf_ctx* ctx);

/* ---- programs (circuit templates) ---- */
int qf_program_create(qf_ctx* ctx, int n_qubits, int n_ops, const qf_op* ops,
                      const double* mats /* [n_mats][4][4][2] or NULL */, int n_mats,
                      int n_params, int precision, qf_program** out);
/* Optional start state (Circuit::initial_state, circuit.hpp:58), 2^n complex128. */
int qf_program_set_initial_state(qf_program* prog, const double* amps);
int qf_program_destroy(qf_program* prog);
/* Schedule introspection: number of fused tile sweeps of the forward and
 * adjoint passes, and tile bits used. */
/* Development: copies the context's psi (which = 0) or lambda (1) work buffer
 * (state-major [B_chunk][2^n]) into `dst` (device or host memory). */
int qf_debug_copy_state(qf_ctx* ctx, int which, void* dst, size_t bytes);
int qf_program_info(const qf_program* prog, int* fwd_sweeps, int* bwd_sweeps,
                    int* fwd_tile_bits, int* bwd_tile_bits);

/* Specialised-kernel status: by default every program's sweeps are compiled
 * into straight-line sm_100a kernels (NVRTC, cached on disk under
 * $QF_JIT_CACHE or ~/.cache/qforge_b200); QF_JIT=0 selects the generic AOT
 * kernels, QF_JIT=2 makes a failed specialisation an error. */
int qf_program_jit_status(const qf_program* prog, int* active, int* compiled, int* cached,
                          double* seconds, const char** error);

/* Host-only introspection (no GPU needed): the compiled schedule as JSON
 * {"n":..,"passes":{"fwd"|"bwd":{"k","R","n_taps","sweeps":[{"tile_bits",
 * "tap_begin","phases":[{"reg_bits","ops":[[dev_kind,gate,tap],..]}]}],
 * "taps":[[slot,coef],..]}}} (needed = bytes incl. NUL), and an NVRTC
 * compile of every specialised kernel of the program for sm_100a. */
int qf_plan_describe(int n_qubits, int n_ops, const qf_op* ops, const double* mats, int n_mats,
                     int n_params, int precision, char* buf, size_t buflen, size_t* needed);
int qf_jit_compile_check(int n_qubits, int n_ops, const qf_op* ops, const double* mats,
                         int n_mats, int n_params, int precision, int* kernels);
/* Host-only: NVRTC compile of the specialised H|psi> kernel of a Pauli sum
 * (codes/weights as qf_observable_create); *compiled = 0 when the sum is above
 * the specialisation limit and the generic kernel would be used. */
int qf_jit_hpsi_check(int n_qubits, int n_terms, const int8_t* codes, const double* w_re, const double* w_im,
                      int precision, int* compiled);

/* ---- observables (Pauli sums) ---- */
/* codes: [n_terms][n_qubits], 0=I 1=X 2=Y 3=Z (pauli.hpp:11-17). */
int qf_observable_create(qf_ctx* ctx, int n_qubits, int n_terms, const int8_t* codes,
                         const double* w_re, const double* w_im, qf_observable** out);
int qf_observable_destroy(qf_observable* obs);
/* Multi-GPU split of qf_energy_grad_batch: QF_SHARD_BATCH (default) gives each
 * rank a contiguous block of parameter sets; QF_SHARD_TERMS gives every rank the
 * whole batch and a contiguous block of Hamiltonian terms (single large state):
 * energies and gradients are linear in H, so the all-reduce sums the parts. */
enum qf_shard { QF_SHARD_BATCH = 0, QF_SHARD_TERMS = 1 };
int qf_observable_set_sharding(qf_observable* obs, int mode);

/* ---- evaluation (host buffers, synchronous) ---- */
/* run(): amps_out = U(theta)|init>, 2^n complex128 interleaved.
 * guard_log2 reproduces run()'s memory guard (circuit.cpp:305-307). */
int qf_run_state(qf_ctx* ctx, const qf_program* prog, const double* theta, int guard_log2,
                 double* amps_out);
/* expectation_pauli(run(theta), obs) as complex (re, im). */
int qf_expectation(qf_ctx* ctx, const qf_program* prog, const qf_observable* obs,
                   const double* theta, double* out_re_im);
/* energies[b] = Re<psi(theta_b)|H|psi(theta_b)>, grads[b][p] = dE/dtheta_p by the
 * adjoint method (grads may be NULL for energies only).  thetas: [batch][n_params].
 * With a communicator attached, all ranks pass the same full batch; each rank
 * evaluates its share and every rank receives the full result. */
int qf_energy_grad_batch(qf_ctx* ctx, const qf_program* prog, const qf_observable* obs,
                         int batch, const double* thetas, double* energies, double* grads);
/* The exact contribution rank `rank` of `world` makes to qf_energy_grad_batch
 * before the all-reduce (zero rows outside its batch block, or its term block's
 * partial sums), with no communicator: the multi-GPU split replayed on one GPU
 * (summing the parts over ranks reproduces the collective's result). */
/* The multi-GPU partition rule (batch rows or Hamiltonian terms): rank r of p
 * owns [count r / p, count (r + 1) / p).  Host-only (no device needed). */
int qf_shard_range(int64_t count, int rank, int world, int64_t* begin, int64_t* end);
int qf_energy_grad_batch_partial(qf_ctx* ctx, const qf_program* prog, const qf_observable* obs,
                                 int batch, const double* thetas, int rank, int world,
                                 double* energies, double* grads);

/* pauli_sum_to_coo (reference src/pauli.cpp:89-153): the Pauli sum as a canonical
 * sparse matrix (row-major, ascending columns, duplicates summed per flip mask,
 * exact zeros dropped), complex128 values [nnz][2].  Call with NULL outputs to
 * get nnz, then with buffers of capacity >= nnz (device pointers when
 * device_buffers != 0).  n_qubits > n_guard -> QF_EINVAL (reference guard 26). */
int qf_pauli_sum_to_coo(qf_ctx* ctx, const qf_observable* obs, int n_guard, int device_buffers,
                        int64_t* rows, int64_t* cols, double* vals, int64_t capacity,
                        int64_t* nnz);

/* energy(ansatz, theta, SparseCOO) (reference variational.cpp:45-52 with the
 * COO matvec of sparse.cpp:44-51): for each of `batch` parameter rows, the
 * forward state psi and E = Re(psi^dagger H psi) over the canonical triplets
 * (rows/cols int64, vals interleaved complex128; host arrays, or device
 * pointers when coo_on_device).  dim must be 2^n ("energy: Hamiltonian
 * dimension mismatch").  Deterministic (fixed-order reductions). */
int qf_sparse_energy(qf_ctx* ctx, const qf_program* prog, int batch, const double* thetas, int64_t dim,
                     int64_t nnz, const int64_t* rows, const int64_t* cols, const double* vals, int coo_on_device,
                     double* energies);

/* Trajectory workload (reference experiments.cpp:210-250, exp_mipt_haar): for
 * each of `trajectories` streams RngStream(seed).split(trajectories)[t], depth
 * brickwork layers of haar_su4 gates on (i, i+1), i = layer % 2, 2, ..., each
 * qubit measured with probability p (measure_collapse, circuit.cpp:391-429),
 * then entropies[t] = subsystem_entropy(psi, {0 .. n/2 - 1}) in bits.  Gates run
 * as batched sweeps with per-trajectory matrices, measurements as batched
 * histogram / collapse passes; the entropy spectrum is rho = A^H A (cuBLAS
 * batched ZGEMM, loaded at run time) reduced by our own batched Householder
 * tridiagonalisation + Sturm bisection kernels (eig.cu, double precision).
 * n in [2, 20], p in [0, 1], trajectories >= 1.
 * n_measurements (optional) receives the total number of collapses. */
int qf_mipt_haar(qf_ctx* ctx, int n, int depth, double p, int trajectories, uint64_t seed, int precision,
                 double* entropies, long long* n_measurements);

/* apply_local_unitary (reference circuit.cpp:78-176) on a host complex128 state
 * (2^n interleaved re/im, in place): U row-major 2^k x 2^k complex128 on
 * wires[0..k) (wires[0] = most significant local bit), 1 <= k <= 13 distinct
 * wires.  One copy in, one kernel, one copy out (no program is built). */
int qf_apply_unitary(qf_ctx* ctx, int n, double* state, int k, const int* wires, const double* u);

/* Eigenvalues (ascending) of `batch` Hermitian m x m matrices a[b] (host,
 * column-major complex128 as interleaved doubles, both triangles), through the
 * device kernels the MIPT entropy uses (m <= 2048).  Exposed for testing. */
int qf_hermitian_eigvals(qf_ctx* ctx, int m, int batch, const double* a, double* w);

/* Classical-shadow snapshots (reference shadows.cpp:50-85): the state of `prep`
 * (at theta) rotated, per snapshot r, into bases[r][0..n) (1 = X, 2 = Y, 3 = Z;
 * basis_rotation, shadows.cpp:33-44) and sampled once by inverse CDF with u[r]
 * (the reference draws u[r] = rng.split(m)[r].uniform()); outcomes[r][q] =
 * bit of qubit q (0 = most significant).  Snapshots run as one batched sweep
 * pass with per-snapshot matrices plus a chunked sampling pass. */
int qf_shadow_snapshots(qf_ctx* ctx, const qf_program* prep, const double* theta, int m, const int8_t* bases,
                        const double* u, int8_t* outcomes);

/* Monte-Carlo noise trajectories (reference noise.cpp:162-197, mc_trajectory),
 * batched: `trajectories` runs of one constant circuit (ops with slot = -1;
 * angles in offset) from |0..0> or `init`.  After op j the channels
 * op_chan[op_chan_ptr[j] .. op_chan_ptr[j+1]) fire in order; channel c's Kraus
 * operators are kraus[chan_kraus_ptr[c] .. chan_kraus_ptr[c+1]) (each 4x4x2
 * doubles, top-left D x D used, D = 2^wires of op j).  Trajectory t consumes the
 * uniforms u[t][0 .. n_apps), n_apps = op_chan_ptr[n_ops], one per application:
 * branch k is picked by u * sum_k p_k against the running sum of
 * p_k = ||K_k psi||^2, psi <- K psi / sqrt(p), log_prob += log(p/acc) + log(acc).
 * Outputs (each optional): states [t][2^n][2], log_probs [t], and with obs the
 * energies Re<psi_t|H|psi_t> in expvals [t]. */
int qf_noise_trajectories(qf_ctx* ctx, int n_qubits, int n_ops, const qf_op* ops, const double* mats, int n_mats,
                          const int* op_chan_ptr, const int* op_chan, const int* chan_kraus_ptr, const double* kraus,
                          const double* init, int trajectories, const double* u, int precision, double* states,
                          double* log_probs, qf_observable* obs, double* expvals);

/* ---- evaluation on device-resident buffers (stream-ordered, no host sync) ----
 * d_thetas [batch][P], d_energies [batch], d_grads [batch][P] (may be NULL), all
 * float64 device pointers.  With a communicator attached every rank passes the
 * full batch and receives the full result, as for qf_energy_grad_batch (the
 * rank's share, one NCCL all-reduce on the context stream). */
int qf_energy_grad_batch_device(qf_ctx* ctx, const qf_program* prog,
                                const qf_observable* obs, int batch,
                                const double* d_thetas, double* d_energies,
                                double* d_grads);
/* vqe_run (reference src/variational.cpp:103-143) with theta, the Adam moments
 * and the energy traces resident on the device: `steps` x (batched energy +
 * gradient, Adam(beta1 0.9, beta2 0.999, eps 1e-8)), then the final energies.
 * theta0 / final_thetas: [batch][P] host; traces: [batch][steps + 1] host
 * (trace[s] = energy before update s, the last entry the final energy);
 * best = first strict minimum of the final energies.  grad_mode: the reference's
 * GradMode (parameter shift / finite differences as one batched evaluation of
 * the 2P shifted sets per step) or the adjoint method. */
enum qf_grad_mode { QF_GRAD_PARAMETER_SHIFT = 0, QF_GRAD_FINITE_DIFF = 1, QF_GRAD_ADJOINT = 2 };
int qf_vqe_run(qf_ctx* ctx, const qf_program* prog, const qf_observable* obs, int batch,
               const double* theta0, int steps, double lr, int grad_mode, double fd_step,
               double* traces, double* final_thetas, double* best_energy, int* best_index);
/* Adam (variational.cpp:83-101) over batch x P device arrays, t = step count after
 * this update (1-based). */
int qf_adam_step_device(qf_ctx* ctx, int batch, int n_params, double* d_theta,
                        double* d_m, double* d_v, const double* d_grad, int t, double lr,
                        double beta1, double beta2, double eps);

/* ---- instrumentation (bench.py) ---- */
/* Counters accumulated since the last qf_ctx_reset_stats: kernel launches (total
 * and per class), algorithmic HBM bytes per class and, when timing is enabled,
 * device time per class from CUDA events recorded on the context stream
 * (resolved lazily, no syncs inside evaluation calls).  Classes: 0 = forward
 * sweeps, 1 = H|psi> / energy, 2 = adjoint sweeps, 3 = reductions. */
int qf_ctx_set_timing(qf_ctx* ctx, int enabled);  /* 0 off, 1 per class, 2 + per launch */
/* Per-launch device times (timing level 2): launch id (forward sweep i, 1000 =
 * H|psi>, 2000 + i = adjoint sweep i), accumulated ms and launch count; *n = the
 * number of ids (entries beyond cap are counted but not written). */
/* Canonical algorithmic flops per class since the last reset (SURVEY.md 8(d):
 * 14 per dense one-qubit gate and amplitude, 6 per diagonal gate, 8 per tap
 * inner product and per Hamiltonian term; adjoint gates count twice). */
int qf_ctx_flops(qf_ctx* ctx, double* flops_by_class /* [4] */);
int qf_ctx_launch_times(qf_ctx* ctx, int cap, int* ids, double* ms, long long* counts, int* n);
int qf_ctx_reset_stats(qf_ctx* ctx);
int qf_ctx_stats(qf_ctx* ctx, long long* launches, long long* launches_by_class /* [4] */,
                 double* ms_by_class /* [4] */, double* bytes_by_class /* [4] */);

#ifdef __cplusplus
}
#endif

#endif /* QFORGE_B200_H */
