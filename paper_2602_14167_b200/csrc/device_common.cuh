// device_common.cuh -- device helpers shared by the AOT interpreter kernels
// (sweep_impl.cuh) and the NVRTC-specialised sweep kernels (jit.cpp).  Must stay
// compilable by NVRTC: no standard-library includes.
#pragma once
#include "plan.h"

namespace qfb {

template <typename RT> struct CxT;
template <> struct CxT<float> { using T = float2; };
template <> struct CxT<double> { using T = double2; };

// a*b + acc (complex), FMA chains
template <typename V> __device__ __forceinline__ V cfma(V a, V b, V acc) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
    V r;
    r.x = a.x * b.x;
    r.x = fma(-a.y, b.y, r.x);
    r.y = a.x * b.y;
    r.y = fma(a.y, b.x, r.y);
    return r;
}
// Im(conj(u) v), Re(conj(u) v)
template <typename V> __device__ __forceinline__ auto imcv(V u, V v) { return fma(u.x, v.y, -u.y * v.x); }
template <typename V> __device__ __forceinline__ auto recv(V u, V v) { return fma(u.x, v.x, u.y * v.y); }

// XOR-fold swizzle of a tile-local amplitude index (linear over GF(2)); W bits
// select the shared-memory bank group (16 x 8B for c64, 8 x 16B for c128).
template <int W> __device__ __forceinline__ uint32_t swz(uint32_t p) {
    uint32_t x = p >> W, f = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f ^= x;
        x >>= W;
    }
    return p ^ (f & ((1u << W) - 1));
}

__device__ __forceinline__ unsigned lane_mask(int T) { return T >= 32 ? 0xffffffffu : ((1u << T) - 1); }

template <typename RT>
__device__ __forceinline__ void tap_store(RT v, double* stap, int tap, int nwarps, int T) {
    const unsigned m = lane_mask(T);
    for (int o = (T >= 32 ? 16 : T / 2); o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
    if ((threadIdx.x & 31) == 0) stap[tap * nwarps + (threadIdx.x >> 5)] = (double)v;
}

// ---------------------------------------------------------------------------
// gate matrices (computed per CTA from theta in double, circuit.cpp:202-302)
// ---------------------------------------------------------------------------
template <typename V, bool ADJ>
__device__ __forceinline__ void put_c(V* out, int o, double re, double im) {
    V r;
    r.x = re;
    r.y = ADJ ? -im : im;
    out[o] = r;
}

// Writes the op's matrix block (the adjoint for the backward pass).  Layouts:
// G1/R1: m00 m01 m10 m11; RX: (c, s) of [[c, -i s], [-i s, c]]; D1: d0 d1;
// D2: d00 d01 d10 d11; G2: row-major 4x4.
template <typename V, bool ADJ>
__device__ void build_matrix(const DevOp& op, const DevGate& g, const double* th,
                             const double* cmats, V* out) {
    const double p = g.slot >= 0 ? g.coef * th[g.slot] + g.offset : g.offset;
    double s, c;
    sincos(0.5 * p, &s, &c);
    const double isq = 0.70710678118654752440;  // 1/sqrt(2), circuit.cpp:205
    switch (g.kind) {
        case GK_H:  // self-adjoint
            put_c<V, false>(out, 0, isq, 0); put_c<V, false>(out, 1, isq, 0);
            put_c<V, false>(out, 2, isq, 0); put_c<V, false>(out, 3, -isq, 0);
            return;
        case GK_RY:
            if (op.kind == DK_RS) {  // shear form: t = tan(phi/2) with |t| <= 1, sign folded as a global phase
                const double sg = ADJ ? -s : s;
                if (c >= 0) {
                    put_c<V, false>(out, 0, sg / (1.0 + c), sg);
                    put_c<V, false>(out, 1, 1.0, 0.0);
                } else {
                    put_c<V, false>(out, 0, -sg / (1.0 - c), -sg);
                    put_c<V, false>(out, 1, -1.0, 0.0);
                }
                return;
            }
            // [[c, -s], [s, c]]; adjoint = transpose
            put_c<V, false>(out, 0, c, 0); put_c<V, false>(out, 1, ADJ ? s : -s, 0);
            put_c<V, false>(out, 2, ADJ ? -s : s, 0); put_c<V, false>(out, 3, c, 0);
            return;
        case GK_RX:
            put_c<V, false>(out, 0, c, ADJ ? -s : s);
            return;
        case GK_Y:  // [[0, -i], [i, 0]], self-adjoint
            put_c<V, false>(out, 0, 0, 0); put_c<V, false>(out, 1, 0, -1);
            put_c<V, false>(out, 2, 0, 1); put_c<V, false>(out, 3, 0, 0);
            return;
        case GK_Z: put_c<V, ADJ>(out, 0, 1, 0); put_c<V, ADJ>(out, 1, -1, 0); return;
        case GK_S: put_c<V, ADJ>(out, 0, 1, 0); put_c<V, ADJ>(out, 1, 0, 1); return;
        case GK_RZ: put_c<V, ADJ>(out, 0, c, -s); put_c<V, ADJ>(out, 1, c, s); return;
        case GK_RZZ:
            put_c<V, ADJ>(out, 0, c, -s); put_c<V, ADJ>(out, 1, c, s);
            put_c<V, ADJ>(out, 2, c, s); put_c<V, ADJ>(out, 3, c, -s);
            return;
        case GK_CZ:
            put_c<V, ADJ>(out, 0, 1, 0); put_c<V, ADJ>(out, 1, 1, 0);
            put_c<V, ADJ>(out, 2, 1, 0); put_c<V, ADJ>(out, 3, -1, 0);
            return;
        case GK_SU4:
        case GK_UNITARY: {
            const double* m = cmats + 32 * (size_t)g.mat;  // row-major 4x4 complex
#define QF_M(r, cc) m[2 * ((r) * 4 + (cc))], m[2 * ((r) * 4 + (cc)) + 1]
            switch (op.kind) {
                case DK_G1: case DK_R1:
                    put_c<V, ADJ>(out, 0, QF_M(0, 0));
                    put_c<V, ADJ>(out, 1, ADJ ? m[2 * 4] : m[2], ADJ ? m[2 * 4 + 1] : m[3]);
                    put_c<V, ADJ>(out, 2, ADJ ? m[2] : m[2 * 4], ADJ ? m[3] : m[2 * 4 + 1]);
                    put_c<V, ADJ>(out, 3, QF_M(1, 1));
                    return;
                case DK_D1:
                    put_c<V, ADJ>(out, 0, QF_M(0, 0)); put_c<V, ADJ>(out, 1, QF_M(1, 1));
                    return;
                case DK_D2:
                    put_c<V, ADJ>(out, 0, QF_M(0, 0)); put_c<V, ADJ>(out, 1, QF_M(1, 1));
                    put_c<V, ADJ>(out, 2, QF_M(2, 2)); put_c<V, ADJ>(out, 3, QF_M(3, 3));
                    return;
                case DK_G2:
                    for (int r = 0; r < 4; ++r)
                        for (int cc = 0; cc < 4; ++cc) {
                            const int sr = ADJ ? cc : r, sc = ADJ ? r : cc;
                            put_c<V, ADJ>(out, r * 4 + cc, QF_M(sr, sc));
                        }
                    return;
                default: return;
            }
#undef QF_M
        }
        default: return;
    }
}

}  // namespace qfb
