// jit_helpers.cuh -- device helpers used by the NVRTC-specialised sweep kernels
// generated in jit.cpp.  The generator emits straight-line code over named
// register variables (x0..x31, y0..y31): gates act on explicit amplitude pairs,
// so permutation gates (x, cx with an in-register control) cost nothing -- the
// generator renames registers instead of moving data.  NVRTC-safe (no includes).
#pragma once
#include "device_common.cuh"

namespace qfb {

__device__ __forceinline__ uint32_t pdep_u32(uint32_t t, uint32_t m) {
    uint32_t r = 0;
    while (m) {
        const uint32_t low = m & (0u - m);
        if (t & 1) r |= low;
        t >>= 1;
        m ^= low;
    }
    return r;
}

template <typename V> __device__ __forceinline__ V mk_basis(bool one) {
    V v;
    v.x = one ? 1 : 0;
    v.y = 0;
    return v;
}

// ---- amplitude arithmetic.  complex64 uses the sm_100 packed FP32 pipe
// (FFMA2 / FMUL2 with scalar-broadcast and swapped-lane operands): a complex
// multiply is 2 instructions instead of 4.  complex128 stays scalar (DFMA).

__device__ __forceinline__ float2 swp(float2 a) { return make_float2(a.y, a.x); }

// QF_NOPACK: the same arithmetic with scalar FP32 instructions (3-register FFMA)
// instead of the packed FFMA2/FMUL2 forms (A/B of the two FP32 issue paths).
#ifdef QF_NOPACK
__device__ __forceinline__ float2 qf_ffma2(float2 a, float2 b, float2 c) {
    return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}
__device__ __forceinline__ float2 qf_fmul2(float2 a, float2 b) { return make_float2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float2 qf_fadd2(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
#else
__device__ __forceinline__ float2 qf_ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 qf_fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 qf_fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
#endif


// a * d (complex)
__device__ __forceinline__ float2 jcmul(float2 a, float2 d) {
    return qf_ffma2(swp(a), make_float2(-d.y, d.y), qf_fmul2(a, make_float2(d.x, d.x)));
}
__device__ __forceinline__ double2 jcmul(double2 a, double2 d) { return cmul(a, d); }
// acc + a * d (complex)
__device__ __forceinline__ float2 jcfma(float2 a, float2 d, float2 acc) {
    return qf_ffma2(swp(a), make_float2(-d.y, d.y), qf_ffma2(a, make_float2(d.x, d.x), acc));
}
__device__ __forceinline__ double2 jcfma(double2 a, double2 d, double2 acc) { return cfma(d, a, acc); }

// real 2x2 [[m0, m1], [m2, m3]] (real parts) on (a0, a1)
__device__ __forceinline__ void jr1(float2& a0, float2& a1, float2 m0, float2 m1, float2 m2, float2 m3) {
    const float2 t0 = a0, t1 = a1;
    a0 = qf_ffma2(t1, make_float2(m1.x, m1.x), qf_fmul2(t0, make_float2(m0.x, m0.x)));
    a1 = qf_ffma2(t1, make_float2(m3.x, m3.x), qf_fmul2(t0, make_float2(m2.x, m2.x)));
}
__device__ __forceinline__ void jr1(double2& a0, double2& a1, double2 m0, double2 m1, double2 m2, double2 m3) {
    const double2 t0 = a0, t1 = a1;
    a0.x = fma(m1.x, t1.x, m0.x * t0.x);
    a0.y = fma(m1.x, t1.y, m0.x * t0.y);
    a1.x = fma(m3.x, t1.x, m2.x * t0.x);
    a1.y = fma(m3.x, t1.y, m2.x * t0.y);
}
// general complex 2x2
template <typename V> __device__ __forceinline__ void jg1(V& a0, V& a1, V m0, V m1, V m2, V m3) {
    const V t0 = a0, t1 = a1;
    a0 = jcfma(t1, m1, jcmul(t0, m0));
    a1 = jcfma(t1, m3, jcmul(t0, m2));
}
// [[c, -i s], [-i s, c]] with m0 = (c, s):  a0' = c a0 + s (a1.y, -a1.x)
__device__ __forceinline__ void jrx(float2& a0, float2& a1, float2 m0) {
    const float2 t0 = a0, t1 = a1;
    const float2 cc = make_float2(m0.x, m0.x), ss = make_float2(m0.y, -m0.y);
    a0 = qf_ffma2(swp(t1), ss, qf_fmul2(t0, cc));
    a1 = qf_ffma2(swp(t0), ss, qf_fmul2(t1, cc));
}
__device__ __forceinline__ void jrx(double2& a0, double2& a1, double2 m0) {
    const double2 t0 = a0, t1 = a1;
    a0.x = fma(m0.y, t1.y, m0.x * t0.x);
    a0.y = fma(-m0.y, t1.x, m0.x * t0.y);
    a1.x = fma(m0.y, t0.y, m0.x * t1.x);
    a1.y = fma(-m0.y, t0.x, m0.x * t1.y);
}
// rotation [[c, -s], [s, c]] (up to a global sign) as three shears, m0 = (t, s)
__device__ __forceinline__ void jrs(float2& a0, float2& a1, float2 m0) {
    const float2 mt = make_float2(-m0.x, -m0.x), ms = make_float2(m0.y, m0.y);
    a0 = qf_ffma2(a1, mt, a0);
    a1 = qf_ffma2(a0, ms, a1);
    a0 = qf_ffma2(a1, mt, a0);
}
__device__ __forceinline__ void jrs(double2& a0, double2& a1, double2 m0) {
    a0.x = fma(-m0.x, a1.x, a0.x);
    a0.y = fma(-m0.x, a1.y, a0.y);
    a1.x = fma(m0.y, a0.x, a1.x);
    a1.y = fma(m0.y, a0.y, a1.y);
    a0.x = fma(-m0.x, a1.x, a0.x);
    a0.y = fma(-m0.x, a1.y, a0.y);
}
// packed tap products (c64): lanes (u.x v.x, u.y v.y) sum to Re(conj(u) v);
// lanes (u.x v.y, u.y v.x) differ to Im(conj(u) v)
__device__ __forceinline__ float2 jre2(float2 u, float2 v) { return qf_fmul2(u, v); }
__device__ __forceinline__ float2 jre2a(float2 u, float2 v, float2 acc) { return qf_ffma2(u, v, acc); }
__device__ __forceinline__ float2 jim2(float2 u, float2 v) { return qf_fmul2(u, swp(v)); }
__device__ __forceinline__ float2 jim2a(float2 u, float2 v, float2 acc) { return qf_ffma2(u, swp(v), acc); }
__device__ __forceinline__ float2 jadd2(float2 a, float2 b) { return qf_fadd2(a, b); }
__device__ __forceinline__ float2 jsub2(float2 a, float2 b) { return qf_fadd2(a, make_float2(-b.x, -b.y)); }
// acc + k v and acc + i k v (k real) for the specialised H|psi> kernels
__device__ __forceinline__ float2 jaxpy(float k, float2 v, float2 acc) { return qf_ffma2(make_float2(k, k), v, acc); }
__device__ __forceinline__ double2 jaxpy(double k, double2 v, double2 acc) {
    return make_double2(fma(k, v.x, acc.x), fma(k, v.y, acc.y));
}
__device__ __forceinline__ float2 jiaxpy(float k, float2 v, float2 acc) {
    return qf_ffma2(make_float2(-k, k), swp(v), acc);
}
__device__ __forceinline__ double2 jiaxpy(double k, double2 v, double2 acc) {
    return make_double2(fma(-k, v.y, acc.x), fma(k, v.x, acc.y));
}
template <typename V> __device__ __forceinline__ void jcswap(V& a, V& b, bool c) {
    const V t0 = a, t1 = b;
    a = c ? t1 : t0;
    b = c ? t0 : t1;
}
// dense 4x4 (row-major m[16]) on (a0, a1, a2, a3) = local basis 00, 01, 10, 11
template <typename V> __device__ __forceinline__ void jg2(V& a0, V& a1, V& a2, V& a3, const V* m) {
    const V v0 = a0, v1 = a1, v2 = a2, v3 = a3;
    a0 = jcfma(v3, m[3], jcfma(v2, m[2], jcfma(v1, m[1], jcmul(v0, m[0]))));
    a1 = jcfma(v3, m[7], jcfma(v2, m[6], jcfma(v1, m[5], jcmul(v0, m[4]))));
    a2 = jcfma(v3, m[11], jcfma(v2, m[10], jcfma(v1, m[9], jcmul(v0, m[8]))));
    a3 = jcfma(v3, m[15], jcfma(v2, m[14], jcfma(v1, m[13], jcmul(v0, m[12]))));
}

// cp.async (LDGSTS) of one amplitude into shared memory (8 B for c64, 16 B for c128)
__device__ __forceinline__ void cp_async_v(float2* dst, const float2* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_v(double2* dst, const double2* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Reduce `cnt` staged taps ([cnt][T] per-thread partials in shared memory) in a
// fixed order (deterministic) and write one partial per tap: out[t * stride].
template <typename RT>
__device__ __forceinline__ void tap_flush(const RT* stg, int cnt, int T, double* out, int stride) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (T + 31) >> 5;
    const unsigned m = lane_mask(T);
    for (int t = warp; t < cnt; t += nw) {
        RT acc = 0;
        for (int j = lane; j < T; j += 32) acc += stg[t * T + j];
        for (int o = (T >= 32 ? 16 : T / 2); o > 0; o >>= 1) acc += __shfl_xor_sync(m, acc, o);
        if (lane == 0) out[(size_t)t * stride] = (double)acc;
    }
}

// TMA bulk copy (cp.async.bulk) of a contiguous global range into shared memory,
// completion counted in bytes on an mbarrier (specialised H|psi> partner tiles)
__device__ __forceinline__ void jit_mbar_init(uint64_t* mb) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
__device__ __forceinline__ void jit_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
    const unsigned m = (unsigned)__cvta_generic_to_shared(mb);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(m), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(m)
                 : "memory");
}
__device__ __forceinline__ void jit_mbar_wait(uint64_t* mb, uint32_t parity) {
    const unsigned m = (unsigned)__cvta_generic_to_shared(mb);
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
                     : "=r"(done)
                     : "r"(m), "r"(parity)
                     : "memory");
}

}  // namespace qfb
