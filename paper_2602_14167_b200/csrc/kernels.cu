// kernels.cu -- sm_100a kernels of the batched state-vector VQE engine.
//
// HBM-streaming kernels (no tensor-core work): every sweep reads each state
// tile once from HBM into a swizzled shared-memory tile, applies a fused run of
// gates in register phases, and writes it back once.  See plan.h and DESIGN.md.
//
// Reference behaviour being replaced (paths relative to /root/reference/proj):
//   sweep_kernel<.., false>  <- run(): apply_local_unitary per gate (src/circuit.cpp:78-176,
//                               304-317), gate_matrix conventions (:202-302)
//   hpsi_kernel              <- expectation_pauli (src/circuit.cpp:319-347), extended to
//                               also produce lambda = H|psi> for the adjoint pass
//   sweep_kernel<.., true>   <- gradient() (src/variational.cpp:54-81): parameter shift
//                               replaced by adjoint back-propagation with in-tile taps
//   reduce_kernel / gather   <- the deterministic per-slot result writes of parallel_for
//                               (include/qforge/parallel.hpp:9-10): fixed-order sums, no
//                               float atomics
//   adam_kernel              <- adam_step (src/variational.cpp:83-101)
#include <cuda_runtime.h>

#include "sweep_impl.cuh"

namespace qfb {

// acc + k * s  and  acc + k * i s  (k real); complex64 on the packed FP32 pipe
__device__ __forceinline__ float2 hp_axpy(float k, float2 s, float2 acc) { return __ffma2_rn(make_float2(k, k), s, acc); }
__device__ __forceinline__ double2 hp_axpy(double k, double2 s, double2 acc) {
    return make_double2(fma(k, s.x, acc.x), fma(k, s.y, acc.y));
}
__device__ __forceinline__ float2 hp_iaxpy(float k, float2 s, float2 acc) {
    return __ffma2_rn(make_float2(-k, k), make_float2(s.y, s.x), acc);
}
__device__ __forceinline__ double2 hp_iaxpy(double k, double2 s, double2 acc) {
    return make_double2(fma(-k, s.y, acc.x), fma(k, s.x, acc.y));
}

// Walsh rows: bit i of c_hp_walsh[z] = parity(i & z), i, z < 16
__constant__ uint16_t c_hp_walsh[16] = {0x0000, 0xaaaa, 0xcccc, 0x6666, 0xf0f0, 0x5a5a, 0x3c3c, 0x9696,
                                        0xff00, 0x55aa, 0x33cc, 0x9966, 0x0ff0, 0xa55a, 0xc33c, 0x6996};

// k with its sign flipped when bit i of M is set (sign-bit xor, no select)
__device__ __forceinline__ float hp_sgn(float k, uint32_t M, int i) {
    return __int_as_float(__float_as_int(k) ^ (int)((M << (31 - i)) & 0x80000000u));
}
__device__ __forceinline__ double hp_sgn(double k, uint32_t M, int i) {
    return __hiloint2double(__double2hiint(k) ^ (int)((M << (31 - i)) & 0x80000000u), __double2loint(k));
}

// s with both parts negated when bit i of M is set
__device__ __forceinline__ double2 hp_negv(double2 s, uint32_t M, int i) {
    const int m = (int)((M << (31 - i)) & 0x80000000u);
    return make_double2(__hiloint2double(__double2hiint(s.x) ^ m, __double2loint(s.x)),
                        __hiloint2double(__double2hiint(s.y) ^ m, __double2loint(s.y)));
}

// one off-diagonal term on the NA amplitudes of a thread: slot i reads the
// partner thread's slot i ^ FH (compile-time offsets off sb)
template <int NA, int TPB, int FH, bool IM, typename V, typename RT>
__device__ __forceinline__ void hp_term(V (&acc)[NA], const V* sb, RT k, uint32_t M) {
    constexpr int TT = NA > 1 ? TPB : 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
        const V s = sb[TT * (i ^ FH)];
        const RT ki = hp_sgn(k, M, i);
        acc[i] = IM ? hp_iaxpy(ki, s, acc[i]) : hp_axpy(ki, s, acc[i]);
    }
}

#define QF_HP_CASE(c) \
    case c:           \
        if constexpr (c < NA) hp_term<NA, TPB, c, IM>(acc, sb, k, M); \
        break;
template <int NA, int TPB, bool IM, typename V, typename RT>
__device__ __forceinline__ void hp_term_sw(int fh, V (&acc)[NA], const V* sb, RT k, uint32_t M) {
    switch (fh) {
        QF_HP_CASE(0) QF_HP_CASE(1) QF_HP_CASE(2) QF_HP_CASE(3) QF_HP_CASE(4) QF_HP_CASE(5)
        QF_HP_CASE(6) QF_HP_CASE(7) QF_HP_CASE(8) QF_HP_CASE(9) QF_HP_CASE(10) QF_HP_CASE(11)
        QF_HP_CASE(12) QF_HP_CASE(13) QF_HP_CASE(14) QF_HP_CASE(15)
        default: break;
    }
}
#undef QF_HP_CASE

// the fields of one term the H|psi> loop needs (coefficients already picked by use_imag)
struct HpTerm {
    int32_t kind, yodd;
    uint32_t f_in, z, fz_par;
    double cr, ci;
};
__device__ __forceinline__ HpTerm hp_load_term(const HArgs& a, int t) {
    const DevTerm& d = a.terms[t];
    HpTerm h;
    h.kind = d.kind;
    h.yodd = d.yodd;
    h.f_in = d.f_in;
    h.z = d.z;
    h.fz_par = d.fz_par;
    h.cr = a.use_imag ? d.ci_re : d.c_re;
    h.ci = a.use_imag ? d.ci_im : d.c_im;
    return h;
}

// cp.async of one amplitude into shared memory (8 B c64 via L1, 16 B c128 via L2)
__device__ __forceinline__ void hp_cp_async(float2* dst, const float2* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src) : "memory");
}
__device__ __forceinline__ void hp_cp_async(double2* dst, const double2* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src) : "memory");
}

// TMA bulk copy (cp.async.bulk, sm_90+) of one contiguous partner tile into shared
// memory, completion counted in bytes on an mbarrier
__device__ __forceinline__ void hp_mbar_init(uint64_t* mb) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
__device__ __forceinline__ void hp_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
    const unsigned m = (unsigned)__cvta_generic_to_shared(mb);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(m), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(m)
                 : "memory");
}
__device__ __forceinline__ void hp_mbar_wait(uint64_t* mb, uint32_t parity) {
    const unsigned m = (unsigned)__cvta_generic_to_shared(mb);
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
                     : "=r"(done)
                     : "r"(m), "r"(parity)
                     : "memory");
}

// ---------------------------------------------------------------------------
// lambda = H psi and E = Re<psi|lambda>, output-stationary per tile.  Partner
// tiles (flip groups above the tile) are double-buffered: the next group's tile
// streams in with cp.async while the current group's terms are applied.
// ---------------------------------------------------------------------------
// TPB threads (compile-time, = blockDim.x when NA > 1) x NA amplitudes per tile
template <typename RT, int NA, int TPB, bool SW>
__global__ void __launch_bounds__(TPB, 3) hpsi_kernel(const HArgs a) {
    using V = typename CxT<RT>::T;
    constexpr int kLgT = TPB == 256 ? 8 : TPB == 128 ? 7 : 0;
    static_assert(NA == 1 || kLgT > 0, "hpsi: TPB must be 128 or 256");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    const uint32_t TS = 1u << a.kh;
    V* own = reinterpret_cast<V*>(smem_raw);
    V* const part = own + TS;  // partner buffer(s): part, and part + TS with a.prefetch
    double* red = reinterpret_cast<double*>(own + (a.prefetch ? 3 : 2) * TS);
    const uint32_t tile = blockIdx.x;
    const int b = blockIdx.y;
    const size_t N = size_t(1) << a.n;
    const V* ps = reinterpret_cast<const V*>(a.psi) + (size_t)b * N;
    const uint32_t base = tile << a.kh;

    V acc[NA];  // the own amplitudes stay in shared memory (registers go to occupancy)
    RT dg[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
        const uint32_t p = tid + (uint32_t)T * i;
        own[p] = ps[base + p];
        acc[i].x = acc[i].y = RT(0);
        dg[i] = RT(0);
    }
    auto next_outer = [&](int from) {
        while (from < a.n_groups && a.groups[from].f_out == 0) ++from;
        return from;
    };
    // Partner tiles are contiguous (the tile is the low kh bits), so with a.tma one
    // thread moves each with a single TMA bulk copy on the buffer's mbarrier;
    // otherwise every thread issues cp.async for its amplitudes.
    __shared__ __align__(8) uint64_t mbar[2];
    uint32_t par[2] = {0u, 0u};
    if (a.tma && tid == 0) {
        hp_mbar_init(&mbar[0]);
        hp_mbar_init(&mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    auto prefetch = [&](int gi, V* buf, int slot) {
        const V* pp = ps + (base ^ a.groups[gi].f_out);
        if (a.tma) {
            if (tid == 0) hp_bulk_load(buf, pp, TS * (uint32_t)sizeof(V), &mbar[slot]);
            return;
        }
#pragma unroll
        for (int i = 0; i < NA; ++i) hp_cp_async(buf + tid + T * i, pp + tid + T * i);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int k = 0;  // outer groups seen
    const int first = next_outer(0);
    if (a.tma) __syncthreads();  // barriers initialised before any use
    if (a.prefetch && first < a.n_groups) prefetch(first, part, 0);
    __syncthreads();
    for (int gi = 0; gi < a.n_groups; ++gi) {
        const DevGroup g = a.groups[gi];
        const V* src = own;
        if (g.f_out && a.prefetch) {
            // this group's tile (buffer k & 1) has landed for every thread, and every
            // thread is done with buffer (k + 1) & 1 (the previous outer group)
            if (a.tma) {
                hp_mbar_wait(&mbar[k & 1], par[k & 1]);
                par[k & 1] ^= 1u;
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            }
            __syncthreads();
            const int nn = next_outer(gi + 1);
            if (nn < a.n_groups) prefetch(nn, part + TS * ((k + 1) & 1), (k + 1) & 1);
            src = part + TS * (k & 1);
            ++k;
        } else if (g.f_out) {  // compute-heavy groups: one staged partner tile
            __syncthreads();  // every thread is done with the previous partner tile
            const V* pp = ps + (base ^ g.f_out);
            if (a.tma) {
                if (tid == 0) hp_bulk_load(part, pp, TS * (uint32_t)sizeof(V), &mbar[0]);
                hp_mbar_wait(&mbar[0], par[0]);
                par[0] ^= 1u;
            } else {
#pragma unroll
                for (int i = 0; i < NA; ++i) part[tid + T * i] = pp[tid + T * i];
                __syncthreads();
            }
            src = part;
        }
        if constexpr (!SW) {
            static_assert(sizeof(RT) == 8, "hpsi: the branch-free body is the complex128 one");
            // complex128: one branch-free body for every term kind (diagonal terms
            // are flip-0 terms, the coefficient is complex with one zero part), so
            // consecutive terms interleave their shared-memory loads
#pragma unroll 2
            for (int t = g.term_begin; t < g.term_end; ++t) {
                const HpTerm d = hp_load_term(a, t);
                const uint32_t zlo = d.z & (TS - 1);
                const uint32_t cpar = (__popc(base & d.z) ^ d.fz_par) & 1;
                const uint32_t s0 = (__popc(tid & zlo) ^ cpar) & 1;
                uint32_t M = (NA > 1 ? (uint32_t)c_hp_walsh[(zlo >> kLgT) & (NA - 1)] : 0u) ^ (0u - s0);
                M = d.kind == TK_FLIP ? 0u : M;
                const RT kr = d.yodd ? RT(0) : (RT)d.cr;
                const RT ki = d.yodd ? (RT)d.ci : RT(0);
                const int fh = NA > 1 ? (int)(d.f_in >> kLgT) : 0;
                const V* sb = src + (tid ^ (d.f_in & (uint32_t)(T - 1)));
                constexpr int TT = NA > 1 ? TPB : 0;
#pragma unroll
                for (int i = 0; i < NA; ++i) {
                    const V sv = hp_negv(sb[TT * (i ^ fh)], M, i);
                    acc[i].x = fma(kr, sv.x, fma(-ki, sv.y, acc[i].x));
                    acc[i].y = fma(kr, sv.y, fma(ki, sv.x, acc[i].y));
                }
            }
        } else {
        // complex64: the next term's fields load while this term is applied
        HpTerm nx;
        if (g.term_begin < g.term_end) nx = hp_load_term(a, g.term_begin);
        for (int t = g.term_begin; t < g.term_end; ++t) {
            const HpTerm d = nx;
            if (t + 1 < g.term_end) nx = hp_load_term(a, t + 1);
            const RT cr = (RT)d.cr;
            const RT ci = (RT)d.ci;
            const uint32_t zlo = d.z & (TS - 1);
            const uint32_t cpar = (__popc(base & d.z) ^ d.fz_par) & 1;
            // amplitude i of this thread is p = tid + TPB i, so parity(p & z) =
            // parity(tid & z) ^ parity(i & z_hi): one Walsh row covers all NA signs
            const uint32_t s0 = (__popc(tid & zlo) ^ cpar) & 1;
            uint32_t M = (NA > 1 ? (uint32_t)c_hp_walsh[(zlo >> kLgT) & (NA - 1)] : 0u) ^ (0u - s0);
            if (d.kind == TK_FLIP) M = 0;
            if (d.kind == TK_DIAG) {
#pragma unroll
                for (int i = 0; i < NA; ++i) dg[i] += hp_sgn(cr, M, i);
            } else {
                // partner of amplitude i: thread tid ^ flo, register slot i ^ fh
                const int fh = NA > 1 ? (int)(d.f_in >> kLgT) : 0;
                const V* sb = src + (tid ^ (d.f_in & (uint32_t)(T - 1)));
                if (!d.yodd)  // real coefficient (Re(w) i^y with y even): acc += (+-cr) src
                    hp_term_sw<NA, TPB, false>(fh, acc, sb, cr, M);
                else  // imaginary coefficient (y odd): acc += (+-ci) i src
                    hp_term_sw<NA, TPB, true>(fh, acc, sb, ci, M);
            }
        }
        }
    }
    double e = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
        const V po = own[tid + T * i];
        acc[i].x = fma(dg[i], po.x, acc[i].x);
        acc[i].y = fma(dg[i], po.y, acc[i].y);
        e += (double)po.x * (double)acc[i].x + (double)po.y * (double)acc[i].y;
    }
    if (a.write_lam) {
        V* lm = reinterpret_cast<V*>(a.lam) + (size_t)b * N;
#pragma unroll
        for (int i = 0; i < NA; ++i) lm[base + tid + T * i] = acc[i];
    }
    const unsigned m = lane_mask(T);
    for (int o = (T >= 32 ? 16 : T / 2); o > 0; o >>= 1) e += __shfl_xor_sync(m, e, o);
    const int nwarps = (T + 31) >> 5;
    if ((tid & 31) == 0) red[tid >> 5] = e;
    __syncthreads();
    if (tid == 0) {
        double s = 0;
        for (int w = 0; w < nwarps; ++w) s += red[w];
        a.epart[(size_t)b * gridDim.x + tile] = s;
    }
}

// gate matrices of every op of one pass, once per parameter set (instead of per CTA)
template <typename RT, bool ADJ>
__global__ void mats_kernel(const DevOp* ops, const int* goff, int n_ops, const DevGate* gates,
                            const double* cmats, const double* theta, int P, int batch_offset,
                            typename CxT<RT>::T* out, int stride, int pass_base, size_t cmats_stride) {
    const int b = blockIdx.y;
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n_ops || goff[o] < 0) return;
    const DevOp op = ops[o];
    // cmats_stride > 0: every state has its own constant matrices (trajectories)
    build_matrix<typename CxT<RT>::T, ADJ>(op, gates[op.gate], theta + (size_t)(b + batch_offset) * P,
                                           cmats + (size_t)(b + batch_offset) * cmats_stride,
                                           out + (size_t)b * stride + pass_base + goff[o]);
}

template <typename RT>
__global__ void init_state_kernel(typename CxT<RT>::T* psi, const typename CxT<RT>::T* init, size_t N) {
    const size_t b = blockIdx.y;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x)
        psi[b * N + i] = init[i];
}

// warp per (b, item): fixed-order sum over tiles (deterministic)
__global__ void reduce_kernel(const ReduceArgs a) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int item = blockIdx.x * (blockDim.x >> 5) + w;
    const int b = blockIdx.y;
    if (item >= a.count) return;
    const double* p = a.part + ((size_t)b * a.count + item) * a.tiles;
    double s = 0;
    for (int t = lane; t < a.tiles; t += 32) s += p[t];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) a.out[(size_t)b * a.count + item] = s;
}

__global__ void gather_grads_kernel(const double* tapsum, int n_taps, const int* slot_ptr,
                                    const int* slot_taps, const double* slot_coef, int P,
                                    double* grads) {
    const int b = blockIdx.y;
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= P) return;
    double g = 0;
    for (int k = slot_ptr[s]; k < slot_ptr[s + 1]; ++k)
        g += slot_coef[k] * tapsum[(size_t)b * n_taps + slot_taps[k]];
    grads[(size_t)b * P + s] = g;
}

// adam_step, variational.cpp:83-101 (c1 = 1 - beta1^t, c2 = 1 - beta2^t from the host)
__global__ void adam_kernel(int count, double* theta, double* m, double* v, const double* g,
                            double lr, double b1, double b2, double eps, double c1, double c2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double gi = g[i];
    const double mi = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = b2 * v[i] + (1.0 - b2) * (gi * gi);
    m[i] = mi;
    v[i] = vi;
    const double mhat = mi / c1;
    const double vhat = vi / c2;
    theta[i] -= lr * mhat / (sqrt(vhat) + eps);
}

// parameter-shift / finite-difference batch (variational.cpp:72-79): row
// (b, j, sgn) = theta_b with theta_b[j] += (sgn ? -shift : +shift)
__global__ void shift_thetas_kernel(int B, int P, const double* theta, double shift, double* out) {
    const int64_t total = (int64_t)B * 2 * P * P;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % P);
        const int64_t row = i / P;  // = (b * P + j) * 2 + sgn
        const int sgn = (int)(row & 1);
        const int j = (int)((row >> 1) % P);
        const int64_t b = (row >> 1) / P;
        double t = theta[b * P + k];
        if (k == j) t = sgn ? theta[b * P + k] - shift : theta[b * P + k] + shift;
        out[i] = t;
    }
}

// g[b][j] = (E(b, j, +) - E(b, j, -)) / denom
__global__ void shift_grad_kernel(int B, int P, const double* E, double denom, double* g) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * P) return;
    g[i] = (E[2 * (int64_t)i] - E[2 * (int64_t)i + 1]) / denom;
}

__global__ void convert_kernel(const float2* src, double2* dst, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = make_double2(src[i].x, src[i].y);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
size_t sweep_smem_bytes(int prec, bool bwd, const DevSweep& sw, int max_mat, int max_taps) {
    const size_t vs = prec == QF_C128 ? 16 : 8;
    const size_t TS = size_t(1) << sw.k;
    const int T = 1 << (sw.k - sw.R);
    const int nwarps = (T + 31) / 32;
    size_t bytes = TS * vs * (bwd ? 2 : 1);
    bytes += (size_t)((max_mat + 1) & ~1) * vs;
    bytes += (size_t)((max_taps * nwarps + 1) & ~1) * 8;
    bytes += (size_t)(sw.op_end - sw.op_begin) * sizeof(DevOp);
    bytes += (size_t)sw.n_phases * sizeof(DevPhase);
    return bytes;
}

cudaError_t launch_sweep_f32_fwd(const SweepArgs&, int, size_t, cudaStream_t);
cudaError_t launch_sweep_f32_bwd(const SweepArgs&, int, size_t, cudaStream_t);
cudaError_t launch_sweep_f64_fwd(const SweepArgs&, int, size_t, cudaStream_t);
cudaError_t launch_sweep_f64_bwd(const SweepArgs&, int, size_t, cudaStream_t);

cudaError_t launch_sweep(int prec, bool bwd, const SweepArgs& a, int batch, int max_mat,
                         int max_taps, cudaStream_t s) {
    const size_t smem = sweep_smem_bytes(prec, bwd, a.sw, max_mat, max_taps);
    if (prec == QF_C128)
        return bwd ? launch_sweep_f64_bwd(a, batch, smem, s) : launch_sweep_f64_fwd(a, batch, smem, s);
    return bwd ? launch_sweep_f32_bwd(a, batch, smem, s) : launch_sweep_f32_fwd(a, batch, smem, s);
}

template <typename RT, int NA, int TPB, bool SW>
static cudaError_t launch_hpsi_t(const HArgs& a, int batch, int T, cudaStream_t s) {
    const size_t vs = sizeof(RT) * 2;
    const size_t smem = ((size_t)(a.prefetch ? 3 : 2) << a.kh) * vs + 8 * 8;
    auto kern = hpsi_kernel<RT, NA, TPB, SW>;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    dim3 grid(1u << (a.n - a.kh), batch);
    kern<<<grid, T, smem, s>>>(a);
    return cudaGetLastError();
}

// 16 amplitudes per thread from 2048-amplitude tiles up (the per-term setup is
// amortised over NA amplitudes), 256 threads below
template <typename RT>
static cudaError_t dispatch_hpsi(const HArgs& a, int batch, cudaStream_t s) {
    const int TS = 1 << a.kh;
    // complex128: the branch-free body with runtime slot offsets (C5: 171 ms per
    // launch vs 216 with the dispatch); complex64: the jump-table dispatch with
    // immediate offsets (C4: 2.82 s vs 2.93 branch-free, 3.19 runtime offsets)
    constexpr bool SW = sizeof(RT) == 4;
    static const bool na8 = std::getenv("QF_HPSI_NA8") && std::getenv("QF_HPSI_NA8")[0] == '1';  // development A/B
    if (TS == 2048 && !na8) return launch_hpsi_t<RT, 16, 128, SW>(a, batch, 128, s);
    const int T = TS < 256 ? TS : 256;
    switch (TS / T) {
        case 1: return launch_hpsi_t<RT, 1, 256, SW>(a, batch, T, s);
        case 2: return launch_hpsi_t<RT, 2, 256, SW>(a, batch, T, s);
        case 4: return launch_hpsi_t<RT, 4, 256, SW>(a, batch, T, s);
        case 8: return launch_hpsi_t<RT, 8, 256, SW>(a, batch, T, s);
        case 16: return launch_hpsi_t<RT, 16, 256, SW>(a, batch, T, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_hpsi(int prec, const HArgs& a, int batch, cudaStream_t s) {
    return prec == QF_C128 ? dispatch_hpsi<double>(a, batch, s) : dispatch_hpsi<float>(a, batch, s);
}

cudaError_t launch_mats(int prec, bool adj, const DevOp* ops, const int* goff, int n_ops, const DevGate* gates,
                        const double* cmats, const double* theta, int P, int batch_offset, void* out, int stride,
                        int pass_base, int batch, cudaStream_t s, size_t cmats_stride) {
    if (n_ops == 0) return cudaSuccess;
    dim3 grid((n_ops + 127) / 128, batch);
    if (prec == QF_C128) {
        if (adj) mats_kernel<double, true><<<grid, 128, 0, s>>>(ops, goff, n_ops, gates, cmats, theta, P, batch_offset, (double2*)out, stride, pass_base, cmats_stride);
        else mats_kernel<double, false><<<grid, 128, 0, s>>>(ops, goff, n_ops, gates, cmats, theta, P, batch_offset, (double2*)out, stride, pass_base, cmats_stride);
    } else {
        if (adj) mats_kernel<float, true><<<grid, 128, 0, s>>>(ops, goff, n_ops, gates, cmats, theta, P, batch_offset, (float2*)out, stride, pass_base, cmats_stride);
        else mats_kernel<float, false><<<grid, 128, 0, s>>>(ops, goff, n_ops, gates, cmats, theta, P, batch_offset, (float2*)out, stride, pass_base, cmats_stride);
    }
    return cudaGetLastError();
}

cudaError_t launch_init_state(int prec, void* psi, const void* init, int n, int batch, cudaStream_t s) {
    const size_t N = size_t(1) << n;
    dim3 grid((unsigned)((N + 255) / 256 < 1024 ? (N + 255) / 256 : 1024), batch);
    if (prec == QF_C128)
        init_state_kernel<double><<<grid, 256, 0, s>>>((double2*)psi, (const double2*)init, N);
    else
        init_state_kernel<float><<<grid, 256, 0, s>>>((float2*)psi, (const float2*)init, N);
    return cudaGetLastError();
}

cudaError_t launch_reduce(const ReduceArgs& a, int batch, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    dim3 grid((a.count + 7) / 8, batch);
    reduce_kernel<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_gather_grads(const double* tapsum, int n_taps, const int* slot_ptr,
                                const int* slot_taps, const double* slot_coef, int P, int batch,
                                double* grads, cudaStream_t s) {
    if (P == 0) return cudaSuccess;
    dim3 grid((P + 127) / 128, batch);
    gather_grads_kernel<<<grid, 128, 0, s>>>(tapsum, n_taps, slot_ptr, slot_taps, slot_coef, P, grads);
    return cudaGetLastError();
}

cudaError_t launch_adam(int count, double* theta, double* m, double* v, const double* g, double lr,
                        double b1, double b2, double eps, double c1, double c2, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    adam_kernel<<<(count + 255) / 256, 256, 0, s>>>(count, theta, m, v, g, lr, b1, b2, eps, c1, c2);
    return cudaGetLastError();
}

cudaError_t launch_shift_thetas(int B, int P, const double* theta, double shift, double* out, cudaStream_t s) {
    if (B == 0 || P == 0) return cudaSuccess;
    shift_thetas_kernel<<<1184, 256, 0, s>>>(B, P, theta, shift, out);
    return cudaGetLastError();
}

cudaError_t launch_shift_grad(int B, int P, const double* E, double denom, double* g, cudaStream_t s) {
    if (B == 0 || P == 0) return cudaSuccess;
    shift_grad_kernel<<<(B * P + 255) / 256, 256, 0, s>>>(B, P, E, denom, g);
    return cudaGetLastError();
}

cudaError_t launch_convert_state(int prec, const void* src, double* dst, int64_t count, cudaStream_t s) {
    if (prec == QF_C128)
        return cudaMemcpyAsync(dst, src, (size_t)count * 16, cudaMemcpyDeviceToDevice, s);
    convert_kernel<<<1024, 256, 0, s>>>((const float2*)src, (double2*)dst, count);
    return cudaGetLastError();
}

}  // namespace qfb
