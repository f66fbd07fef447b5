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

// real 2x2 [[m0, m1], [m2, m3]] (real parts) on (a0, a1)
template <typename V> __device__ __forceinline__ void jr1(V& a0, V& a1, V m0, V m1, V m2, V m3) {
    const V t0 = a0, t1 = a1;
    a0.x = fma(m1.x, t1.x, m0.x * t0.x);
    a0.y = fma(m1.x, t1.y, m0.x * t0.y);
    a1.x = fma(m3.x, t1.x, m2.x * t0.x);
    a1.y = fma(m3.x, t1.y, m2.x * t0.y);
}
// general complex 2x2
template <typename V> __device__ __forceinline__ void jg1(V& a0, V& a1, V m0, V m1, V m2, V m3) {
    const V t0 = a0, t1 = a1;
    a0 = cfma(m1, t1, cmul(m0, t0));
    a1 = cfma(m3, t1, cmul(m2, t0));
}
// [[c, -i s], [-i s, c]] with m0 = (c, s)
template <typename V> __device__ __forceinline__ void jrx(V& a0, V& a1, V m0) {
    const V t0 = a0, t1 = a1;
    a0.x = fma(m0.y, t1.y, m0.x * t0.x);
    a0.y = fma(-m0.y, t1.x, m0.x * t0.y);
    a1.x = fma(m0.y, t0.y, m0.x * t1.x);
    a1.y = fma(-m0.y, t0.x, m0.x * t1.y);
}
template <typename V> __device__ __forceinline__ void jcswap(V& a, V& b, bool c) {
    const V t0 = a, t1 = b;
    a = c ? t1 : t0;
    b = c ? t0 : t1;
}
// dense 4x4 (row-major m[16]) on (a0, a1, a2, a3) = local basis 00, 01, 10, 11
template <typename V> __device__ __forceinline__ void jg2(V& a0, V& a1, V& a2, V& a3, const V* m) {
    const V v0 = a0, v1 = a1, v2 = a2, v3 = a3;
    a0 = cfma(m[3], v3, cfma(m[2], v2, cfma(m[1], v1, cmul(m[0], v0))));
    a1 = cfma(m[7], v3, cfma(m[6], v2, cfma(m[5], v1, cmul(m[4], v0))));
    a2 = cfma(m[11], v3, cfma(m[10], v2, cfma(m[9], v1, cmul(m[8], v0))));
    a3 = cfma(m[15], v3, cfma(m[14], v2, cfma(m[13], v1, cmul(m[12], v0))));
}

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

}  // namespace qfb
