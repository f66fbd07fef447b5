/*
 * qforge_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C99, complex double) of the reference qforge hot path,
 * used as the parity checker for the CUDA engine.  Only tests/, the smoke()
 * check in __graft_entry__.py and the cpu_baseline / --impl reference legs of
 * bench.py may load this library.  The product path never links or calls it.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 */
#ifndef QFORGE_ORACLE_H
#define QFORGE_ORACLE_H

#include <complex.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Gate enum, same order as include/qforge/circuit.hpp:14-23 */
enum {
    QO_H = 0, QO_X, QO_Y, QO_Z, QO_S,
    QO_RX, QO_RY, QO_RZ, QO_RZZ,
    QO_CX, QO_CZ,
    QO_SU4, QO_CSUM, QO_SUBSPACE_RY, QO_SUBSPACE_RZ,
    QO_UNITARY
};

/* One op of a parameter template: param = coef * theta[slot] + offset when
 * slot >= 0, else offset.  mat indexes a table of 4x4 (row-major) complex
 * matrices for QO_UNITARY / QO_SU4 (2x2 gates use the top-left 2x2 corner of
 * the row-major 4x4, same layout as the product's qf_program_create). */
typedef struct qo_op {
    int32_t kind;
    int32_t q0;
    int32_t q1;   /* -1 for 1-qubit gates */
    int32_t slot; /* -1: constant */
    double coef;
    double offset;
    int32_t mat;  /* -1 unless QO_UNITARY/QO_SU4 */
    int32_t pad;
} qo_op;

typedef struct qo_rng {
    uint64_t seed, stream, counter;
    int32_t have_spare;
    int32_t pad;
    double spare;
} qo_rng;

/* ---- RngStream (include/qforge/rng.hpp:12-85) ---- */
void qo_rng_init(qo_rng* r, uint64_t seed, uint64_t stream);
uint64_t qo_rng_next_u64(qo_rng* r);
double qo_rng_uniform(qo_rng* r);
uint64_t qo_rng_uniform_below(qo_rng* r, uint64_t bound);
double qo_rng_normal(qo_rng* r);
void qo_rng_split_child(const qo_rng* r, uint64_t i, qo_rng* child);

/* ---- engine (src/circuit.cpp) ---- */
/* returns 0 ok, -1 invalid argument (message in qo_last_error) */
int qo_run(int n, int n_ops, const qo_op* ops, const double complex* mats,
           const double* theta, const double complex* init, int guard_log2,
           double complex* out);
int qo_apply_local_unitary(int n, double complex* psi, const double complex* u,
                           int k, const int* wires);
int qo_gate_matrix(const qo_op* op, const double complex* mats, const double* theta,
                   double complex* u /* 16 */, int* dim);
int qo_expectation_pauli(int n, const double complex* psi, int n_terms,
                         const double* w_re, const double* w_im, const int8_t* codes,
                         double complex* out);

/* ---- variational (src/variational.cpp) ---- */
typedef struct qo_ansatz {
    int n;
    int n_params;
    int n_ops;
    const qo_op* ops;
    const double complex* mats;
    const double complex* init; /* nullable initial state */
    int guard_log2;
} qo_ansatz;

typedef struct qo_hamil {
    int n;
    int n_terms;
    const double* w_re;
    const double* w_im;
    const int8_t* codes; /* [n_terms][n] */
} qo_hamil;

int qo_energy(const qo_ansatz* a, const double* theta, const qo_hamil* h, double* e);
/* mode 0 = parameter_shift, 1 = finite_diff, 2 = adjoint (new math, CPU) */
int qo_gradient(const qo_ansatz* a, const double* theta, const qo_hamil* h, int mode,
                double fd_step, int workers, double* grad);
void qo_adam_step(double* m, double* v, int* t, double* theta, const double* grad,
                  int p, double lr, double beta1, double beta2, double eps);
/* traces: [B][steps+1]; final_thetas: [B][P] */
int qo_vqe_run(const qo_ansatz* a, int batch, const double* theta0, const qo_hamil* h,
               int steps, double lr, int mode, int workers, double* traces,
               double* final_thetas, double* best_energy, int* best_index);
/* batched energy + gradient, batch-parallel over workers (bench CPU baseline) */
int qo_energy_grad_batch(const qo_ansatz* a, int batch, const double* thetas,
                         const qo_hamil* h, int mode, int workers, double* energies,
                         double* grads);

/* ---- model builders (src/pauli.cpp:181-203, lattice.cpp:89-170 chain,
 *      tests/helpers.hpp:52-63) ---- codes out: [T][n] int8, weights re/im */
int qo_chain_edges(int n, int pbc, int* edges /* [2*max] */);
int qo_tfim_terms(int n, int pbc, double g, double* w_re, double* w_im, int8_t* codes);
int qo_heisenberg_terms(int n, int pbc, double jx, double jy, double jz, double* w_re,
                        double* w_im, int8_t* codes);
void qo_random_pauli_sum(int n, int terms, qo_rng* rng, int real_weights, double* w_re,
                         double* w_im, int8_t* codes);

/* pauli_sum_to_coo (src/pauli.cpp:89-153): returns nnz; with non-NULL outputs
 * (capacity >= nnz) fills canonical row-major triplets. */
long long qo_pauli_sum_to_coo(int n, int n_terms, const double* w_re, const double* w_im,
                              const int8_t* codes, long long* rows, long long* cols,
                              double complex* vals, long long capacity);

/* fixture generation: split gate loops over t threads (bit-identical results) */
void qo_set_inner_threads(int t);

const char* qo_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
