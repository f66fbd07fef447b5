/*
 * qforge_oracle.c -- TEST INFRASTRUCTURE ONLY (see qforge_oracle.h).
 *
 * Line-faithful C99 restatement of the reference qforge hot path.  Built with
 * gcc -O2 and no -ffast-math / -march, like proj/src/CMakeLists.txt:8, so the
 * complex-double arithmetic rounds the way the reference's std::complex code
 * does.  The reference itself cannot be compiled here (Eigen and vendor/ are
 * absent), see DESIGN.md "Oracle".
 */
#include "qforge_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

/* Intra-state threading for fixture generation at n = 26/30 (default 1 = the
 * reference's single-threaded loops).  Only loops whose iterations write
 * disjoint amplitudes with the reference's per-element arithmetic are split,
 * and per-term expectation sums are still accumulated in term order, so the
 * results are bit-identical to the sequential restatement. */
static int g_inner = 1;
void qo_set_inner_threads(int t) { g_inner = t < 1 ? 1 : t; }

typedef void (*range_fn)(void* ctx, int64_t b, int64_t e);
typedef struct { range_fn fn; void* ctx; int64_t b, e; } range_job;
static void* range_worker(void* p) {
    range_job* j = (range_job*)p;
    j->fn(j->ctx, j->b, j->e);
    return NULL;
}
/* fn over [0, n) in g_inner contiguous chunks (sequential below 2^16 items) */
static void par_range(int64_t n, range_fn fn, void* ctx) {
    int w = g_inner;
    if (w <= 1 || n < ((int64_t)1 << 16)) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t th[256];
    range_job jobs[256];
    if (w > 256) w = 256;
    for (int i = 0; i < w; ++i) {
        jobs[i] = (range_job){fn, ctx, n * i / w, n * (i + 1) / w};
        pthread_create(&th[i], NULL, range_worker, &jobs[i]);
    }
    for (int i = 0; i < w; ++i) pthread_join(th[i], NULL);
}

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}
const char* qo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* RngStream: include/qforge/rng.hpp:12-85                                   */
/* ------------------------------------------------------------------------ */
static uint64_t mix_(uint64_t z) { /* rng.hpp:71-75 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static uint64_t key_(const qo_rng* r) { /* rng.hpp:76-78 */
    return mix_(r->seed ^ 0xA0761D6478BD642FULL) ^ mix_(r->stream ^ 0xE7037ED1A0B428DBULL);
}
void qo_rng_init(qo_rng* r, uint64_t seed, uint64_t stream) {
    memset(r, 0, sizeof *r);
    r->seed = seed;
    r->stream = stream;
}
uint64_t qo_rng_next_u64(qo_rng* r) { /* rng.hpp:21-27 */
    uint64_t z = key_(r) + r->counter * 0x9E3779B97F4A7C15ULL;
    ++r->counter;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
double qo_rng_uniform(qo_rng* r) { /* rng.hpp:30-32 */
    return (double)(qo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}
uint64_t qo_rng_uniform_below(qo_rng* r, uint64_t bound) { /* rng.hpp:35-41 */
    if (bound <= 1) return 0;
    uint64_t limit = ~0ULL - (~0ULL % bound);
    uint64_t v;
    do { v = qo_rng_next_u64(r); } while (v >= limit);
    return v % bound;
}
double qo_rng_normal(qo_rng* r) { /* rng.hpp:44-57 */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = qo_rng_uniform(r);
    double u2 = qo_rng_uniform(r);
    if (u1 < 1e-300) u1 = 1e-300;
    double rr = sqrt(-2.0 * log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    r->spare = rr * sin(a);
    r->have_spare = 1;
    return rr * cos(a);
}
void qo_rng_split_child(const qo_rng* r, uint64_t i, qo_rng* child) { /* rng.hpp:60-68 */
    uint64_t c = mix_(r->stream ^ mix_(0xD1B54A32D192ED03ULL + i));
    qo_rng_init(child, r->seed, c);
}

/* ------------------------------------------------------------------------ */
/* gate_matrix: src/circuit.cpp:202-302 (qubit gates)                        */
/* ------------------------------------------------------------------------ */
static double op_param(const qo_op* op, const double* theta) {
    if (op->slot >= 0) return op->coef * theta[op->slot] + op->offset;
    return op->offset;
}

int qo_gate_matrix(const qo_op* op, const double complex* mats, const double* theta,
                   double complex* u, int* dim) {
    const double isq = 1.0 / sqrt(2.0);
    for (int i = 0; i < 16; ++i) u[i] = 0.0;
    switch (op->kind) {
        case QO_H: *dim = 2; u[0] = isq; u[1] = isq; u[2] = isq; u[3] = -isq; return 0;
        case QO_X: *dim = 2; u[1] = 1; u[2] = 1; return 0;
        case QO_Y: *dim = 2; u[1] = CMPLX(0, -1); u[2] = CMPLX(0, 1); return 0;
        case QO_Z: *dim = 2; u[0] = 1; u[3] = -1; return 0;
        case QO_S: *dim = 2; u[0] = 1; u[3] = CMPLX(0, 1); return 0;
        case QO_RX: { /* circuit.cpp:220-224 */
            double t = op_param(op, theta);
            double complex c = cos(0.5 * t), s = CMPLX(0.0, -sin(0.5 * t));
            *dim = 2; u[0] = c; u[1] = s; u[2] = s; u[3] = c; return 0;
        }
        case QO_RY: { /* circuit.cpp:225-229 */
            double t = op_param(op, theta);
            double c = cos(0.5 * t), s = sin(0.5 * t);
            *dim = 2; u[0] = c; u[1] = -s; u[2] = s; u[3] = c; return 0;
        }
        case QO_RZ: { /* circuit.cpp:230-236, std::polar(1, x) = (cos x, sin x) */
            double t = op_param(op, theta);
            *dim = 2;
            u[0] = CMPLX(cos(-0.5 * t), sin(-0.5 * t));
            u[3] = CMPLX(cos(0.5 * t), sin(0.5 * t));
            return 0;
        }
        case QO_RZZ: { /* circuit.cpp:237-243 */
            double t = op_param(op, theta);
            double complex em = CMPLX(cos(-0.5 * t), sin(-0.5 * t));
            double complex ep = CMPLX(cos(0.5 * t), sin(0.5 * t));
            *dim = 4; u[0] = em; u[5] = ep; u[10] = ep; u[15] = em; return 0;
        }
        case QO_CX: *dim = 4; u[0] = 1; u[5] = 1; u[11] = 1; u[14] = 1; return 0;
        case QO_CZ: *dim = 4; u[0] = 1; u[5] = 1; u[10] = 1; u[15] = -1; return 0;
        case QO_SU4:
        case QO_UNITARY: {
            if (op->mat < 0 || !mats) return fail("gate_matrix: missing matrix");
            *dim = op->q1 >= 0 ? 4 : 2;
            const double complex* m = mats + 16 * (size_t)op->mat;
            if (*dim == 4) memcpy(u, m, 16 * sizeof(double complex));
            else { u[0] = m[0]; u[1] = m[1]; u[2] = m[4]; u[3] = m[5]; }
            return 0;
        }
        default: return fail("gate_matrix: unsupported gate for the qubit hot path");
    }
}

/* ------------------------------------------------------------------------ */
/* apply_local_unitary: src/circuit.cpp:78-176 (d == 2)                       */
/* ------------------------------------------------------------------------ */
typedef struct {
    double complex* a;
    const double complex* u;
    int64_t dk, s0, s1;
    int k;
    int64_t ws[8];
} alu_ctx;

static void alu_diag(void* p, int64_t b, int64_t e) { /* :96-107 */
    alu_ctx* c = (alu_ctx*)p;
    for (int64_t idx = b; idx < e; ++idx) {
        int64_t loc = 0;
        for (int i = 0; i < c->k; ++i) loc = (loc << 1) | ((idx / c->ws[i]) & 1);
        c->a[idx] *= c->u[loc * c->dk + loc];
    }
}

/* pair index j -> lo = j with a zero inserted at stride s (the :112-121 loop nest, flattened) */
static void alu_1q(void* p, int64_t b, int64_t e) {
    alu_ctx* c = (alu_ctx*)p;
    const int64_t s = c->s0;
    const double complex u00 = c->u[0], u01 = c->u[1], u10 = c->u[2], u11 = c->u[3];
    double complex* a = c->a;
    for (int64_t j = b; j < e; ++j) {
        const int64_t lo = ((j & ~(s - 1)) << 1) | (j & (s - 1));
        double complex a0 = a[lo], a1 = a[lo + s];
        a[lo] = u00 * a0 + u01 * a1;
        a[lo + s] = u10 * a0 + u11 * a1;
    }
}

static void alu_2q(void* p, int64_t b, int64_t e) { /* :128-144, flattened */
    alu_ctx* c = (alu_ctx*)p;
    const int64_t s0 = c->s0, s1 = c->s1;
    const int64_t hibit = s0 > s1 ? s0 : s1, lobit = s0 < s1 ? s0 : s1;
    double complex m[4][4];
    for (int r = 0; r < 4; ++r)
        for (int q = 0; q < 4; ++q) m[r][q] = c->u[r * 4 + q];
    double complex* a = c->a;
    for (int64_t j = b; j < e; ++j) {
        int64_t x = ((j & ~(lobit - 1)) << 1) | (j & (lobit - 1));
        const int64_t base = ((x & ~(hibit - 1)) << 1) | (x & (hibit - 1));
        double complex v[4] = {a[base], a[base + s1], a[base + s0], a[base + s0 + s1]};
        for (int r = 0; r < 4; ++r) {
            a[base + (r >> 1) * s0 + (r & 1) * s1] =
                m[r][0] * v[0] + m[r][1] * v[1] + m[r][2] * v[2] + m[r][3] * v[3];
        }
    }
}

int qo_apply_local_unitary(int n, double complex* a, const double complex* u, int k,
                           const int* wires) {
    const int64_t dk = (int64_t)1 << k;
    for (int i = 0; i < k; ++i)
        if (wires[i] < 0 || wires[i] >= n) return fail("apply_local_unitary: wire out of range");
    int64_t stride[64];
    for (int i = 0; i < n; ++i) stride[i] = (int64_t)1 << (n - 1 - i); /* :86-87 */
    const int64_t dim = (int64_t)1 << n;
    alu_ctx c;
    c.a = a;
    c.u = u;
    c.dk = dk;
    c.k = k;
#define U(r, c) u[(r) * dk + (c)]
    if (k <= 8) { /* :90-108 diagonal fast path, exact-zero test */
        int diagonal = 1;
        for (int64_t r = 0; r < dk && diagonal; ++r)
            for (int64_t q = 0; q < dk && diagonal; ++q)
                if (r != q && U(r, q) != 0.0) diagonal = 0;
        if (diagonal) {
            for (int i = 0; i < k; ++i) c.ws[i] = stride[wires[i]];
            par_range(dim, alu_diag, &c);
            return 0;
        }
    }
#undef U
    if (k == 1) { /* :109-122 */
        c.s0 = stride[wires[0]];
        par_range(dim / 2, alu_1q, &c);
        return 0;
    }
    if (k == 2) { /* :123-145 */
        c.s0 = stride[wires[0]];
        c.s1 = stride[wires[1]];
        par_range(dim / 4, alu_2q, &c);
        return 0;
    }
    return fail("apply_local_unitary: only 1- and 2-qubit gates on the hot path");
}

static int op_wires(const qo_op* op, int* wires) {
    wires[0] = op->q0;
    if (op->q1 >= 0) {
        wires[1] = op->q1;
        return 2;
    }
    return 1;
}

/* run: src/circuit.cpp:304-317 plus the Circuit::gate validation :178-186 */
int qo_run(int n, int n_ops, const qo_op* ops, const double complex* mats,
           const double* theta, const double complex* init, int guard_log2,
           double complex* out) {
    if (n < 1 || n > 40) return fail("run: bad qubit count");
    double dim = pow(2.0, n);
    if (!(dim <= pow(2.0, (double)guard_log2)))
        return fail("run: state dimension exceeds memory guard");
    const int64_t N = (int64_t)1 << n;
    if (init) memcpy(out, init, (size_t)N * sizeof(double complex));
    else {
        memset(out, 0, (size_t)N * sizeof(double complex));
        out[0] = 1.0;
    }
    for (int i = 0; i < n_ops; ++i) {
        int wires[2];
        int k = op_wires(&ops[i], wires);
        for (int w = 0; w < k; ++w)
            if (wires[w] < 0 || wires[w] >= n) return fail("Circuit: wire out of range");
        if (k == 2 && wires[0] == wires[1]) return fail("Circuit: duplicate wires");
        double p = op_param(&ops[i], theta);
        if (!isfinite(p)) return fail("Circuit: non-finite parameter");
        double complex u[16];
        int d;
        if (qo_gate_matrix(&ops[i], mats, theta, u, &d)) return -1;
        if ((d == 4) != (k == 2)) return fail("apply_local_unitary: wrong gate size");
        if (qo_apply_local_unitary(n, out, u, k, wires)) return -1;
    }
    return 0;
}

/* expectation_pauli: src/circuit.cpp:319-347.  Each term's sum runs over s in
 * the reference order; with inner threads the terms are spread over threads and
 * the per-term sums are still added to acc in term order (bit-identical). */
typedef struct {
    int n;
    const double complex* psi;
    const double* w_re;
    const double* w_im;
    const int8_t* codes;
    double complex* sums;
} ex_ctx;

static double complex term_sum(int n, const double complex* psi, double wr, double wi,
                               const int8_t* code) {
    static const double complex ipowt[4] = {1.0, CMPLX(0, 1), -1.0, CMPLX(0, -1)};
    const int64_t dim = (int64_t)1 << n;
    uint64_t flip = 0, zmask = 0;
    int ycount = 0;
    for (int i = 0; i < n; ++i) {
        uint64_t bit = 1ULL << (n - 1 - i);
        switch (code[i]) {
            case 1: flip |= bit; break;
            case 2: flip |= bit; zmask |= bit; ++ycount; break;
            case 3: zmask |= bit; break;
            default: break;
        }
    }
    double complex base = CMPLX(wr, wi) * ipowt[ycount & 3];
    double complex sum = 0.0;
    for (int64_t s = 0; s < dim; ++s) {
        double complex v = base;
        if (__builtin_parityll((uint64_t)s & zmask)) v = -v;
        sum += conj(psi[s ^ (int64_t)flip]) * v * psi[s];
    }
    return sum;
}

static void ex_terms(void* p, int64_t b, int64_t e) {
    ex_ctx* c = (ex_ctx*)p;
    for (int64_t t = b; t < e; ++t)
        c->sums[t] = term_sum(c->n, c->psi, c->w_re[t], c->w_im[t], c->codes + (size_t)t * c->n);
}

int qo_expectation_pauli(int n, const double complex* psi, int n_terms,
                         const double* w_re, const double* w_im, const int8_t* codes,
                         double complex* out) {
    double complex acc = 0.0;
    if (g_inner > 1 && n >= 16 && n_terms > 1) {
        double complex* sums = malloc((size_t)n_terms * sizeof(double complex));
        ex_ctx c = {n, psi, w_re, w_im, codes, sums};
        int w = g_inner < n_terms ? g_inner : n_terms;
        pthread_t th[256];
        range_job jobs[256];
        if (w > 256) w = 256;
        for (int i = 0; i < w; ++i) {
            jobs[i] = (range_job){ex_terms, &c, (int64_t)n_terms * i / w, (int64_t)n_terms * (i + 1) / w};
            pthread_create(&th[i], NULL, range_worker, &jobs[i]);
        }
        for (int i = 0; i < w; ++i) pthread_join(th[i], NULL);
        for (int t = 0; t < n_terms; ++t) acc += sums[t];
        free(sums);
    } else {
        for (int t = 0; t < n_terms; ++t)
            acc += term_sum(n, psi, w_re[t], w_im[t], codes + (size_t)t * n);
    }
    *out = acc;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* variational: src/variational.cpp                                          */
/* ------------------------------------------------------------------------ */
int qo_energy(const qo_ansatz* a, const double* theta, const qo_hamil* h, double* e) {
    /* variational.cpp:38-43 */
    if (h->n != a->n) return fail("expectation_pauli: size mismatch");
    const int64_t N = (int64_t)1 << a->n;
    double complex* psi = malloc((size_t)N * sizeof(double complex));
    if (!psi) return fail("energy: out of memory");
    int rc = qo_run(a->n, a->n_ops, a->ops, a->mats, theta, a->init, a->guard_log2, psi);
    if (rc == 0) {
        double complex v;
        qo_expectation_pauli(a->n, psi, h->n_terms, h->w_re, h->w_im, h->codes, &v);
        *e = creal(v);
    }
    free(psi);
    return rc;
}

/* static-stride thread pool: include/qforge/parallel.hpp:11-26 */
typedef void (*pf_fn)(void* ctx, size_t i);
typedef struct { pf_fn fn; void* ctx; size_t n, w, workers; } pf_job;
static void* pf_worker(void* p) {
    pf_job* j = (pf_job*)p;
    for (size_t i = j->w; i < j->n; i += j->workers) j->fn(j->ctx, i);
    return NULL;
}
static void parallel_for(size_t n, size_t workers, pf_fn fn, void* ctx) {
    if (workers <= 1 || n <= 1) {
        for (size_t i = 0; i < n; ++i) fn(ctx, i);
        return;
    }
    if (workers > n) workers = n;
    pthread_t* th = malloc(workers * sizeof(pthread_t));
    pf_job* jobs = malloc(workers * sizeof(pf_job));
    for (size_t w = 0; w < workers; ++w) {
        jobs[w] = (pf_job){fn, ctx, n, w, workers};
        pthread_create(&th[w], NULL, pf_worker, &jobs[w]);
    }
    for (size_t w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
    free(jobs);
}

typedef struct {
    const qo_ansatz* a;
    const double* theta;
    const qo_hamil* h;
    double shift, denom;
    double* grad;
    int err;
} grad_ctx;

static void grad_one(void* p, size_t j) { /* variational.cpp:72-79 */
    grad_ctx* c = (grad_ctx*)p;
    int P = c->a->n_params;
    double* t = malloc((size_t)(P > 0 ? P : 1) * sizeof(double));
    memcpy(t, c->theta, (size_t)P * sizeof(double));
    double ep = 0, em = 0;
    t[j] = c->theta[j] + c->shift;
    if (qo_energy(c->a, t, c->h, &ep)) c->err = 1;
    t[j] = c->theta[j] - c->shift;
    if (qo_energy(c->a, t, c->h, &em)) c->err = 1;
    c->grad[j] = (ep - em) / c->denom;
    free(t);
}

/* generator of a shift-eligible rotation: 1 = X, 2 = Y, 3 = Z, 4 = ZZ */
static int rotation_generator(int kind) {
    switch (kind) {
        case QO_RX: return 1;
        case QO_RY: return 2;
        case QO_RZ: return 3;
        case QO_RZZ: return 4;
        default: return 0;
    }
}

/* Adjoint gradient (NEW math: the reference has none, variational.hpp:30).
 * U_j = exp(-i p_j G_j / 2), p_j = coef_j theta[slot_j] + offset_j:
 *   dE/dtheta_s = sum_{j: slot_j = s} coef_j * Im <lambda_j| G_j |psi_j>,
 * with psi_j the state after gate j and lambda_j = U_{j+1}^+ ... U_G^+ H psi.
 * H uses Re(w) only: Re<psi|H|psi> depends on the Hermitian part alone. */
typedef struct {
    const double complex* in;
    double complex* out;
    double complex base;
    uint64_t flip, zmask;
    int64_t b0, b1;
    int gen;
    const double complex* lam;
    double* part;
    int64_t chunk;
} gen_ctx;

static void ps_term(void* p, int64_t b, int64_t e) {
    gen_ctx* c = (gen_ctx*)p;
    for (int64_t s = b; s < e; ++s) {
        double complex v = c->base;
        if (__builtin_parityll((uint64_t)s & c->zmask)) v = -v;
        c->out[s ^ (int64_t)c->flip] += v * c->in[s];
    }
}

static void apply_pauli_sum(int n, const qo_hamil* h, const double complex* psi,
                            double complex* out) {
    const int64_t dim = (int64_t)1 << n;
    static const double complex ipowt[4] = {1.0, CMPLX(0, 1), -1.0, CMPLX(0, -1)};
    memset(out, 0, (size_t)dim * sizeof(double complex));
    for (int t = 0; t < h->n_terms; ++t) {
        uint64_t flip = 0, zmask = 0;
        int y = 0;
        for (int i = 0; i < n; ++i) {
            uint64_t bit = 1ULL << (n - 1 - i);
            int c = h->codes[(size_t)t * n + i];
            if (c == 1) flip |= bit;
            if (c == 2) { flip |= bit; zmask |= bit; ++y; }
            if (c == 3) zmask |= bit;
        }
        /* (P psi)[s ^ flip] = base * (-1)^{popc(s & z)} psi[s]: s -> s ^ flip is a bijection */
        gen_ctx c = {psi, out, h->w_re[t] * ipowt[y & 3], flip, zmask, 0, 0, 0, NULL, NULL, 0};
        par_range(dim, ps_term, &c);
    }
}

static void gen_apply(void* p, int64_t b, int64_t e) {
    gen_ctx* c = (gen_ctx*)p;
    const double complex* in = c->in;
    double complex* out = c->out;
    for (int64_t s = b; s < e; ++s) {
        int bit0 = (s & c->b0) != 0;
        switch (c->gen) {
            case 1: out[s] = in[s ^ c->b0]; break;
            case 2: out[s] = (bit0 ? CMPLX(0, 1) : CMPLX(0, -1)) * in[s ^ c->b0]; break;
            case 3: out[s] = bit0 ? -in[s] : in[s]; break;
            case 4: out[s] = (bit0 ^ ((s & c->b1) != 0)) ? -in[s] : in[s]; break;
        }
    }
}

static void apply_generator(int n, int gen, int q0, int q1, const double complex* in,
                            double complex* out) {
    const int64_t dim = (int64_t)1 << n;
    gen_ctx c = {in, out, 0, 0, 0, (int64_t)1 << (n - 1 - q0), q1 >= 0 ? (int64_t)1 << (n - 1 - q1) : 0,
                 gen, NULL, NULL, 0};
    par_range(dim, gen_apply, &c);
}

/* Im <lambda|tmp>, summed in fixed chunks of 2^16 (new math, order fixed for any thread count) */
static void im_chunks(void* p, int64_t b, int64_t e) {
    gen_ctx* c = (gen_ctx*)p;
    for (int64_t k = b; k < e; ++k) {
        double im = 0.0;
        for (int64_t s = k * c->chunk; s < (k + 1) * c->chunk; ++s) im += cimag(conj(c->lam[s]) * c->in[s]);
        c->part[k] = im;
    }
}

static double im_inner(int64_t N, const double complex* lam, const double complex* tmp) {
    const int64_t chunk = N < ((int64_t)1 << 16) ? N : ((int64_t)1 << 16);
    const int64_t nc = N / chunk;
    double* part = malloc((size_t)nc * sizeof(double));
    gen_ctx c = {tmp, NULL, 0, 0, 0, 0, 0, 0, lam, part, chunk};
    if (g_inner > 1 && nc >= g_inner) {
        pthread_t th[256];
        range_job jobs[256];
        int w = g_inner > 256 ? 256 : g_inner;
        for (int i = 0; i < w; ++i) {
            jobs[i] = (range_job){im_chunks, &c, nc * i / w, nc * (i + 1) / w};
            pthread_create(&th[i], NULL, range_worker, &jobs[i]);
        }
        for (int i = 0; i < w; ++i) pthread_join(th[i], NULL);
    } else {
        im_chunks(&c, 0, nc);
    }
    double im = 0.0;
    for (int64_t k = 0; k < nc; ++k) im += part[k];
    free(part);
    return im;
}

static int adjoint_gradient(const qo_ansatz* a, const double* theta, const qo_hamil* h,
                            double* grad) {
    const int n = a->n;
    const int64_t N = (int64_t)1 << n;
    double complex* psi = malloc((size_t)N * sizeof(double complex));
    double complex* lam = malloc((size_t)N * sizeof(double complex));
    double complex* tmp = malloc((size_t)N * sizeof(double complex));
    int rc = qo_run(n, a->n_ops, a->ops, a->mats, theta, a->init, a->guard_log2, psi);
    if (rc == 0) {
        apply_pauli_sum(n, h, psi, lam);
        for (int p = 0; p < a->n_params; ++p) grad[p] = 0.0;
        for (int j = a->n_ops - 1; j >= 0; --j) {
            const qo_op* op = &a->ops[j];
            int gen = rotation_generator(op->kind);
            if (op->slot >= 0) {
                if (!gen) { rc = fail("adjoint: parameter feeds a non-rotation gate"); break; }
                apply_generator(n, gen, op->q0, op->q1, psi, tmp);
                const double im = im_inner(N, lam, tmp);
                grad[op->slot] += op->coef * im;
            }
            double complex u[16], ud[16];
            int d, wires[2];
            int k = op_wires(op, wires);
            qo_gate_matrix(op, a->mats, theta, u, &d);
            for (int r = 0; r < d; ++r)
                for (int c = 0; c < d; ++c) ud[r * d + c] = conj(u[c * d + r]);
            qo_apply_local_unitary(n, psi, ud, k, wires);
            qo_apply_local_unitary(n, lam, ud, k, wires);
        }
    }
    free(psi);
    free(lam);
    free(tmp);
    return rc;
}

int qo_gradient(const qo_ansatz* a, const double* theta, const qo_hamil* h, int mode,
                double fd_step, int workers, double* grad) {
    /* variational.cpp:54-81 */
    if (a->n_params < 0) return fail("AnsatzSpec: negative parameter count");
    if (mode == 2) return adjoint_gradient(a, theta, h, grad);
    if (mode == 0) {
        /* shift eligibility: every op fed by a slot must be a +-1/2-eigenvalue rotation */
        for (int i = 0; i < a->n_ops; ++i)
            if (a->ops[i].slot >= 0 && !rotation_generator(a->ops[i].kind))
                return fail("gradient: parameter not shift-eligible, use finite_diff");
    } else if (!(fd_step > 0.0)) {
        return fail("gradient: finite-diff step must be positive");
    }
    grad_ctx c = {a, theta, h, mode == 0 ? M_PI / 2.0 : fd_step,
                  mode == 0 ? 2.0 : 2.0 * fd_step, grad, 0};
    parallel_for((size_t)a->n_params, (size_t)(workers > 1 ? workers : 1), grad_one, &c);
    return c.err ? fail("gradient: energy evaluation failed") : 0;
}

void qo_adam_step(double* m, double* v, int* t, double* theta, const double* grad, int p,
                  double lr, double beta1, double beta2, double eps) {
    /* variational.cpp:83-101 */
    if (*t == 0) {
        for (int i = 0; i < p; ++i) m[i] = v[i] = 0.0;
    }
    ++*t;
    for (int i = 0; i < p; ++i) m[i] = beta1 * m[i] + (1.0 - beta1) * grad[i];
    for (int i = 0; i < p; ++i) v[i] = beta2 * v[i] + (1.0 - beta2) * (grad[i] * grad[i]);
    const double c1 = 1.0 - pow(beta1, *t);
    const double c2 = 1.0 - pow(beta2, *t);
    for (int i = 0; i < p; ++i) {
        double mhat = m[i] / c1;
        double vhat = v[i] / c2;
        theta[i] -= lr * mhat / (sqrt(vhat) + eps);
    }
}

typedef struct {
    const qo_ansatz* a;
    const double* theta0;
    const qo_hamil* h;
    int steps, mode, inner;
    double lr;
    double* traces;
    double* final_thetas;
    int err;
} vqe_ctx;

static void vqe_one(void* p, size_t b) { /* variational.cpp:119-131 */
    vqe_ctx* c = (vqe_ctx*)p;
    const int P = c->a->n_params;
    double* theta = c->final_thetas + b * (size_t)P;
    memcpy(theta, c->theta0 + b * (size_t)P, (size_t)P * sizeof(double));
    size_t bytes = (size_t)(P > 0 ? P : 1) * sizeof(double);
    double *m = malloc(bytes), *v = malloc(bytes), *g = malloc(bytes);
    int t = 0;
    for (int s = 0; s < c->steps; ++s) {
        double e = 0;
        if (qo_energy(c->a, theta, c->h, &e)) c->err = 1;
        c->traces[b * (size_t)(c->steps + 1) + s] = e;
        if (qo_gradient(c->a, theta, c->h, c->mode, 1e-5, c->inner, g)) c->err = 1;
        qo_adam_step(m, v, &t, theta, g, P, c->lr, 0.9, 0.999, 1e-8);
    }
    free(m);
    free(v);
    free(g);
}

int qo_vqe_run(const qo_ansatz* a, int batch, const double* theta0, const qo_hamil* h,
               int steps, double lr, int mode, int workers, double* traces,
               double* final_thetas, double* best_energy, int* best_index) {
    /* variational.cpp:103-143 */
    if (batch < 1) return fail("vqe_run: empty batch");
    if (steps < 1) return fail("vqe_run: steps must be >= 1");
    int w = workers > 1 ? workers : 1;
    int outer = batch < w ? batch : w;
    int inner = w / outer > 1 ? w / outer : 1;
    vqe_ctx c = {a, theta0, h, steps, mode, inner, lr, traces, final_thetas, 0};
    parallel_for((size_t)batch, (size_t)outer, vqe_one, &c);
    if (c.err) return fail("vqe_run: evaluation failed");
    *best_energy = INFINITY;
    *best_index = -1;
    for (int b = 0; b < batch; ++b) {
        double e = 0;
        if (qo_energy(a, final_thetas + (size_t)b * a->n_params, h, &e)) return -1;
        traces[(size_t)b * (steps + 1) + steps] = e;
        if (e < *best_energy) {
            *best_energy = e;
            *best_index = b;
        }
    }
    return 0;
}

typedef struct {
    const qo_ansatz* a;
    const double* thetas;
    const qo_hamil* h;
    int mode, inner;
    double* energies;
    double* grads;
    int err;
} batch_ctx;

static void batch_one(void* p, size_t b) {
    batch_ctx* c = (batch_ctx*)p;
    const size_t P = (size_t)c->a->n_params;
    if (qo_energy(c->a, c->thetas + b * P, c->h, &c->energies[b])) c->err = 1;
    if (c->grads && qo_gradient(c->a, c->thetas + b * P, c->h, c->mode, 1e-5, c->inner,
                                c->grads + b * P))
        c->err = 1;
}

int qo_energy_grad_batch(const qo_ansatz* a, int batch, const double* thetas,
                         const qo_hamil* h, int mode, int workers, double* energies,
                         double* grads) {
    int w = workers > 1 ? workers : 1;
    int outer = batch < w ? batch : w;
    int inner = w / outer > 1 ? w / outer : 1;
    batch_ctx c = {a, thetas, h, mode, inner, energies, grads, 0};
    parallel_for((size_t)batch, (size_t)outer, batch_one, &c);
    return c.err ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* pauli_sum_to_coo: src/pauli.cpp:89-153 (single worker; per-row entries      */
/* sorted by column with a stable insertion sort, duplicates summed in term  */
/* order, exact zeros dropped)                                                */
/* ------------------------------------------------------------------------ */
long long qo_pauli_sum_to_coo(int n, int n_terms, const double* w_re, const double* w_im,
                              const int8_t* codes, long long* rows, long long* cols,
                              double complex* vals, long long capacity) {
    static const double complex ipow[4] = {1.0, CMPLX(0, 1), -1.0, CMPLX(0, -1)};
    if (n < 1) { fail("pauli_sum_to_coo: empty system"); return -1; }
    const uint64_t dim = 1ULL << n;
    uint64_t* flip = malloc(sizeof(uint64_t) * (n_terms + 1));
    uint64_t* zm = malloc(sizeof(uint64_t) * (n_terms + 1));
    double complex* base = malloc(sizeof(double complex) * (n_terms + 1));
    for (int t = 0; t < n_terms; ++t) { /* compile_term, pauli.cpp:61-74 */
        flip[t] = zm[t] = 0;
        int y = 0;
        for (int i = 0; i < n; ++i) {
            uint64_t bit = 1ULL << (n - 1 - i);
            switch (codes[(size_t)t * n + i]) {
                case 1: flip[t] |= bit; break;
                case 2: flip[t] |= bit; zm[t] |= bit; ++y; break;
                case 3: zm[t] |= bit; break;
            }
        }
        base[t] = CMPLX(w_re[t], w_im[t]) * ipow[y & 3];
    }
    uint64_t* ec = malloc(sizeof(uint64_t) * (n_terms + 1));
    double complex* ev = malloc(sizeof(double complex) * (n_terms + 1));
    long long total = 0;
    for (uint64_t row = 0; row < dim; ++row) {
        int m = 0;
        for (int t = 0; t < n_terms; ++t) { /* term_value, pauli.cpp:79-85 */
            uint64_t col = row ^ flip[t];
            double complex v = base[t];
            if (__builtin_parityll(col & zm[t])) v = -v;
            int j = m++;
            while (j > 0 && ec[j - 1] > col) { ec[j] = ec[j - 1]; ev[j] = ev[j - 1]; --j; }
            ec[j] = col;
            ev[j] = v;
        }
        int k = 0;
        while (k < m) {
            double complex v = ev[k];
            int k2 = k + 1;
            while (k2 < m && ec[k2] == ec[k]) v += ev[k2++];
            if (v != 0.0) {
                if (rows && total < capacity) {
                    rows[total] = (long long)row;
                    cols[total] = (long long)ec[k];
                    vals[total] = v;
                }
                ++total;
            }
            k = k2;
        }
    }
    free(flip); free(zm); free(base); free(ec); free(ev);
    return total;
}

/* ------------------------------------------------------------------------ */
/* model builders                                                            */
/* ------------------------------------------------------------------------ */
typedef struct { double d; int i, j; } pair_t;
static int pair_cmp(const void* x, const void* y) { /* lattice.cpp:105-109 */
    const pair_t *a = x, *b = y;
    if (a->d != b->d) return a->d < b->d ? -1 : 1;
    if (a->i != b->i) return a->i < b->i ? -1 : 1;
    return a->j < b->j ? -1 : (a->j > b->j);
}

/* order-1 edges of build_lattice(chain, {n}, {pbc}) (lattice.cpp:29-48, 89-122) */
int qo_chain_edges(int n, int pbc, int* edges) {
    if (n < 1) return fail("build_lattice: size entries must be >= 1");
    if (pbc && n < 3) return fail("build_lattice: periodic dimension needs extent >= 3");
    if (n < 2) return 0;
    size_t np = (size_t)n * (n - 1) / 2, k = 0;
    pair_t* pr = malloc(np * sizeof(pair_t));
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            double d = fabs((double)i - (double)j);
            if (pbc) {
                double best = INFINITY;
                for (int m = -1; m <= 1; ++m) {
                    double s = fabs(((double)i - (double)j) + (double)m * (double)n);
                    if (s < best) best = s;
                }
                d = best;
            }
            pr[k++] = (pair_t){d, i, j};
        }
    qsort(pr, np, sizeof(pair_t), pair_cmp);
    int order = 0, ne = 0;
    double shell = -1.0;
    for (size_t p = 0; p < np; ++p) {
        if (pr[p].d <= 0.0) continue;
        if (shell < 0.0 || pr[p].d > shell * (1.0 + 1e-6)) {
            ++order;
            shell = pr[p].d;
        }
        if (order > 1) break;
        edges[2 * ne] = pr[p].i;
        edges[2 * ne + 1] = pr[p].j;
        ++ne;
    }
    free(pr);
    return ne;
}

int qo_tfim_terms(int n, int pbc, double g, double* w_re, double* w_im, int8_t* codes) {
    /* pauli.cpp:181-189 */
    int* edges = malloc(sizeof(int) * 2 * (size_t)(n * (n > 1 ? n : 1) + 2));
    int ne = qo_chain_edges(n, pbc, edges);
    if (ne < 0) { free(edges); return -1; }
    if (ne == 0) { free(edges); return fail("tfim_terms: lattice has no order-1 edges"); }
    int t = 0;
    for (int e = 0; e < ne; ++e, ++t) {
        memset(codes + (size_t)t * n, 0, (size_t)n);
        codes[(size_t)t * n + edges[2 * e]] = 3;
        codes[(size_t)t * n + edges[2 * e + 1]] = 3;
        w_re[t] = -1.0;
        w_im[t] = 0.0;
    }
    for (int i = 0; i < n; ++i, ++t) {
        memset(codes + (size_t)t * n, 0, (size_t)n);
        codes[(size_t)t * n + i] = 1;
        w_re[t] = -g;
        w_im[t] = 0.0;
    }
    free(edges);
    return t;
}

int qo_heisenberg_terms(int n, int pbc, double jx, double jy, double jz, double* w_re,
                        double* w_im, int8_t* codes) {
    /* pauli.cpp:191-203 */
    int* edges = malloc(sizeof(int) * 2 * (size_t)(n * (n > 1 ? n : 1) + 2));
    int ne = qo_chain_edges(n, pbc, edges);
    if (ne < 0) { free(edges); return -1; }
    if (ne == 0) { free(edges); return fail("heisenberg_terms: lattice has no order-1 edges"); }
    const double js[3] = {jx, jy, jz};
    int t = 0;
    for (int e = 0; e < ne; ++e)
        for (int axis = 0; axis < 3; ++axis) {
            if (js[axis] == 0.0) continue;
            memset(codes + (size_t)t * n, 0, (size_t)n);
            codes[(size_t)t * n + edges[2 * e]] = (int8_t)(axis + 1);
            codes[(size_t)t * n + edges[2 * e + 1]] = (int8_t)(axis + 1);
            w_re[t] = js[axis];
            w_im[t] = 0.0;
            ++t;
        }
    free(edges);
    return t;
}

void qo_random_pauli_sum(int n, int terms, qo_rng* rng, int real_weights, double* w_re,
                         double* w_im, int8_t* codes) {
    /* tests/helpers.hpp:52-63 */
    for (int t = 0; t < terms; ++t) {
        for (int q = 0; q < n; ++q) codes[(size_t)t * n + q] = (int8_t)qo_rng_uniform_below(rng, 4);
        if (real_weights) {
            w_re[t] = qo_rng_normal(rng);
            w_im[t] = 0.0;
        } else {
            /* cplx(rng.normal(), rng.normal()): C++17 leaves argument evaluation
             * order unspecified; gcc on x86-64 evaluates right-to-left, so the
             * imaginary part is drawn first. */
            double im = qo_rng_normal(rng);
            double re = qo_rng_normal(rng);
            w_re[t] = re;
            w_im[t] = im;
        }
    }
}
