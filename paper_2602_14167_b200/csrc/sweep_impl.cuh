// sweep_impl.cuh -- device code of the AOT (interpreter) fused tile sweep
// (included by the per-precision/direction translation units so they compile
// in parallel).  The NVRTC-specialised variant lives in jit.cpp.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "../../include/qforge_b200.h"
#include "device_common.cuh"
#include "kernels.cuh"

namespace qfb {

template <int V_> using IC = std::integral_constant<int, V_>;

template <int R, typename F> __device__ __forceinline__ void with_rb(int rb, F&& f) {
    switch (rb) {
        case 0: f(IC<0>{}); break;
        case 1: if constexpr (R > 1) f(IC<1>{}); break;
        case 2: if constexpr (R > 2) f(IC<2>{}); break;
        case 3: if constexpr (R > 3) f(IC<3>{}); break;
        case 4: if constexpr (R > 4) f(IC<4>{}); break;
        default: break;
    }
}

// ---------------------------------------------------------------------------
// register-resident gate bodies (RB = register bit, compile time)
// ---------------------------------------------------------------------------
template <int RB, int NR, typename V>
__device__ __forceinline__ void k_g1(V* x, V m0, V m1, V m2, V m3) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        V a0 = x[i], a1 = x[j];
        x[i] = cfma(m1, a1, cmul(m0, a0));
        x[j] = cfma(m3, a1, cmul(m2, a0));
    }
}
template <int RB, int NR, typename V, typename RT>
__device__ __forceinline__ void k_r1(V* x, RT r00, RT r01, RT r10, RT r11) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        V a0 = x[i], a1 = x[j];
        x[i].x = fma(r01, a1.x, r00 * a0.x);
        x[i].y = fma(r01, a1.y, r00 * a0.y);
        x[j].x = fma(r11, a1.x, r10 * a0.x);
        x[j].y = fma(r11, a1.y, r10 * a0.y);
    }
}
// [[c, -i s], [-i s, c]]
template <int RB, int NR, typename V, typename RT>
__device__ __forceinline__ void k_rx(V* x, RT c, RT s) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        V a0 = x[i], a1 = x[j];
        x[i].x = fma(s, a1.y, c * a0.x);
        x[i].y = fma(-s, a1.x, c * a0.y);
        x[j].x = fma(s, a0.y, c * a1.x);
        x[j].y = fma(-s, a0.x, c * a1.y);
    }
}
// rotation as three shears: a0 -= t a1; a1 += s a0; a0 -= t a1   (m = (t, s))
template <int RB, int NR, typename V, typename RT>
__device__ __forceinline__ void k_rs(V* x, RT t, RT s) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        V a0 = x[i], a1 = x[j];
        a0.x = fma(-t, a1.x, a0.x);
        a0.y = fma(-t, a1.y, a0.y);
        a1.x = fma(s, a0.x, a1.x);
        a1.y = fma(s, a0.y, a1.y);
        a0.x = fma(-t, a1.x, a0.x);
        a0.y = fma(-t, a1.y, a0.y);
        x[i] = a0;
        x[j] = a1;
    }
}
template <int RB, int NR, typename V> __device__ __forceinline__ void k_x1(V* x) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        V t = x[i];
        x[i] = x[j];
        x[j] = t;
    }
}
// controlled X with the control in registers too: pure register renaming
template <int RB, int CB, int NR, typename V> __device__ __forceinline__ void k_cx_rr(V* x) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if ((i & (1 << RB)) || !(i & (1 << CB))) continue;
        const int j = i | (1 << RB);
        V t = x[i];
        x[i] = x[j];
        x[j] = t;
    }
}
// controlled X with a thread-level control bit: predicated swap
template <int RB, int NR, typename V> __device__ __forceinline__ void k_cx_rt(V* x, bool c) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        V t0 = x[i], t1 = x[j];
        x[i] = c ? t1 : t0;
        x[j] = c ? t0 : t1;
    }
}
template <int RB, int NR, typename V> __device__ __forceinline__ void k_d1(V* x, V d0, V d1) {
#pragma unroll
    for (int i = 0; i < NR; ++i) x[i] = cmul(x[i], (i & (1 << RB)) ? d1 : d0);
}
template <int NR, typename V> __device__ __forceinline__ void k_dc(V* x, V d) {
#pragma unroll
    for (int i = 0; i < NR; ++i) x[i] = cmul(x[i], d);
}
template <int RB0, int RB1, int NR, typename V>
__device__ __forceinline__ void k_d2(V* x, const V* d) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        const int idx = ((i >> RB0) & 1) * 2 + ((i >> RB1) & 1);
        x[i] = cmul(x[i], d[idx]);
    }
}
template <int RB0, int RB1, int NR, typename V>
__device__ __forceinline__ void k_g2(V* x, const V* m) {
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if ((i & (1 << RB0)) || (i & (1 << RB1))) continue;
        int id[4] = {i, i | (1 << RB1), i | (1 << RB0), i | (1 << RB0) | (1 << RB1)};
        V v[4] = {x[id[0]], x[id[1]], x[id[2]], x[id[3]]};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            V acc = cmul(m[r * 4 + 0], v[0]);
            acc = cfma(m[r * 4 + 1], v[1], acc);
            acc = cfma(m[r * 4 + 2], v[2], acc);
            acc = cfma(m[r * 4 + 3], v[3], acc);
            x[id[r]] = acc;
        }
    }
}

// ---- adjoint taps: per-thread partial of Im<lambda|G|psi> (x = psi, y = lambda)
template <int RB, int NR, typename V> __device__ __forceinline__ auto t_x(const V* x, const V* y) {
    decltype(x[0].x) s = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        s += imcv(y[i], x[j]) + imcv(y[j], x[i]);
    }
    return s;
}
// Y|0> = i|1>, Y|1> = -i|0>:  (Y psi)_i = -i psi_j (bit 0), +i psi_i' (bit 1)
template <int RB, int NR, typename V> __device__ __forceinline__ auto t_y(const V* x, const V* y) {
    decltype(x[0].x) s = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << RB)) continue;
        const int j = i | (1 << RB);
        s += recv(y[j], x[i]) - recv(y[i], x[j]);
    }
    return s;
}
template <int RB, int NR, typename V> __device__ __forceinline__ auto t_z(const V* x, const V* y) {
    decltype(x[0].x) s = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        auto v = imcv(y[i], x[i]);
        s += (i & (1 << RB)) ? -v : v;
    }
    return s;
}
template <int RB0, int RB1, int NR, typename V>
__device__ __forceinline__ auto t_zz(const V* x, const V* y) {
    decltype(x[0].x) s = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        auto v = imcv(y[i], x[i]);
        s += (((i >> RB0) ^ (i >> RB1)) & 1) ? -v : v;
    }
    return s;
}
template <int NR, typename V> __device__ __forceinline__ auto t_sum(const V* x, const V* y) {
    decltype(x[0].x) s = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) s += imcv(y[i], x[i]);
    return s;
}


// ---------------------------------------------------------------------------
// one op inside a phase
// ---------------------------------------------------------------------------
template <typename RT, int R, bool BWD, typename V>
__device__ __forceinline__ void apply_op(const DevOp& op, V* x, V* y, uint32_t g_t, const V* smat,
                                         double* stap, int nwarps, int T) {
    constexpr int NR = 1 << R;
    switch (op.kind) {
        case DK_G1: {
            const V m0 = smat[op.moff], m1 = smat[op.moff + 1], m2 = smat[op.moff + 2], m3 = smat[op.moff + 3];
            with_rb<R>(op.rb0, [&](auto B) {
                k_g1<decltype(B)::value, NR>(x, m0, m1, m2, m3);
                if constexpr (BWD) k_g1<decltype(B)::value, NR>(y, m0, m1, m2, m3);
            });
            break;
        }
        case DK_R1: {
            const RT r00 = smat[op.moff].x, r01 = smat[op.moff + 1].x, r10 = smat[op.moff + 2].x,
                     r11 = smat[op.moff + 3].x;
            with_rb<R>(op.rb0, [&](auto B) {
                k_r1<decltype(B)::value, NR>(x, r00, r01, r10, r11);
                if constexpr (BWD) k_r1<decltype(B)::value, NR>(y, r00, r01, r10, r11);
            });
            break;
        }
        case DK_RX: {
            const RT c = smat[op.moff].x, s = smat[op.moff].y;
            with_rb<R>(op.rb0, [&](auto B) {
                k_rx<decltype(B)::value, NR>(x, c, s);
                if constexpr (BWD) k_rx<decltype(B)::value, NR>(y, c, s);
            });
            break;
        }
        case DK_RS: {
            const RT t = smat[op.moff].x, s = smat[op.moff].y;
            with_rb<R>(op.rb0, [&](auto B) {
                k_rs<decltype(B)::value, NR>(x, t, s);
                if constexpr (BWD) k_rs<decltype(B)::value, NR>(y, t, s);
            });
            break;
        }
        case DK_X1:
            with_rb<R>(op.rb0, [&](auto B) {
                k_x1<decltype(B)::value, NR>(x);
                if constexpr (BWD) k_x1<decltype(B)::value, NR>(y);
            });
            break;
        case DK_CX:
            if (op.rb1 >= 0) {
                with_rb<R>(op.rb0, [&](auto B) {
                    with_rb<R>(op.rb1, [&](auto C) {
                        if constexpr (decltype(B)::value != decltype(C)::value) {
                            k_cx_rr<decltype(B)::value, decltype(C)::value, NR>(x);
                            if constexpr (BWD) k_cx_rr<decltype(B)::value, decltype(C)::value, NR>(y);
                        }
                    });
                });
            } else {
                const bool c = (g_t >> op.pos0) & 1;
                with_rb<R>(op.rb0, [&](auto B) {
                    k_cx_rt<decltype(B)::value, NR>(x, c);
                    if constexpr (BWD) k_cx_rt<decltype(B)::value, NR>(y, c);
                });
            }
            break;
        case DK_D1: {
            const V d0 = smat[op.moff], d1 = smat[op.moff + 1];
            if (op.rb0 >= 0) {
                with_rb<R>(op.rb0, [&](auto B) {
                    k_d1<decltype(B)::value, NR>(x, d0, d1);
                    if constexpr (BWD) k_d1<decltype(B)::value, NR>(y, d0, d1);
                });
            } else {
                const V d = ((g_t >> op.pos0) & 1) ? d1 : d0;
                k_dc<NR>(x, d);
                if constexpr (BWD) k_dc<NR>(y, d);
            }
            break;
        }
        case DK_D2: {
            V d[4] = {smat[op.moff], smat[op.moff + 1], smat[op.moff + 2], smat[op.moff + 3]};
            if (op.rb0 >= 0 && op.rb1 >= 0) {
                with_rb<R>(op.rb0, [&](auto B) {
                    with_rb<R>(op.rb1, [&](auto C) {
                        if constexpr (decltype(B)::value != decltype(C)::value) {
                            k_d2<decltype(B)::value, decltype(C)::value, NR>(x, d);
                            if constexpr (BWD) k_d2<decltype(B)::value, decltype(C)::value, NR>(y, d);
                        }
                    });
                });
            } else if (op.rb0 >= 0) {
                const int c1 = (g_t >> op.pos1) & 1;
                const V e0 = d[c1], e1 = d[2 + c1];
                with_rb<R>(op.rb0, [&](auto B) {
                    k_d1<decltype(B)::value, NR>(x, e0, e1);
                    if constexpr (BWD) k_d1<decltype(B)::value, NR>(y, e0, e1);
                });
            } else if (op.rb1 >= 0) {
                const int c0 = (g_t >> op.pos0) & 1;
                const V e0 = d[2 * c0], e1 = d[2 * c0 + 1];
                with_rb<R>(op.rb1, [&](auto B) {
                    k_d1<decltype(B)::value, NR>(x, e0, e1);
                    if constexpr (BWD) k_d1<decltype(B)::value, NR>(y, e0, e1);
                });
            } else {
                const V e = d[((g_t >> op.pos0) & 1) * 2 + ((g_t >> op.pos1) & 1)];
                k_dc<NR>(x, e);
                if constexpr (BWD) k_dc<NR>(y, e);
            }
            break;
        }
        case DK_G2: {
            const V* m = smat + op.moff;
            with_rb<R>(op.rb0, [&](auto B) {
                with_rb<R>(op.rb1, [&](auto C) {
                    if constexpr (decltype(B)::value != decltype(C)::value) {
                        k_g2<decltype(B)::value, decltype(C)::value, NR>(x, m);
                        if constexpr (BWD) k_g2<decltype(B)::value, decltype(C)::value, NR>(y, m);
                    }
                });
            });
            break;
        }
        default:
            if constexpr (BWD) {
                RT v = 0;
                switch (op.kind) {
                    case DK_TX:
                        with_rb<R>(op.rb0, [&](auto B) { v = t_x<decltype(B)::value, NR>(x, y); });
                        break;
                    case DK_TY:
                        with_rb<R>(op.rb0, [&](auto B) { v = t_y<decltype(B)::value, NR>(x, y); });
                        break;
                    case DK_TZ:
                        if (op.rb0 >= 0) {
                            with_rb<R>(op.rb0, [&](auto B) { v = t_z<decltype(B)::value, NR>(x, y); });
                        } else {
                            v = t_sum<NR>(x, y);
                            if ((g_t >> op.pos0) & 1) v = -v;
                        }
                        break;
                    case DK_TZZ:
                        if (op.rb0 >= 0 && op.rb1 >= 0) {
                            with_rb<R>(op.rb0, [&](auto B) {
                                with_rb<R>(op.rb1, [&](auto C) {
                                    if constexpr (decltype(B)::value != decltype(C)::value)
                                        v = t_zz<decltype(B)::value, decltype(C)::value, NR>(x, y);
                                });
                            });
                        } else if (op.rb0 >= 0 || op.rb1 >= 0) {
                            const int rb = op.rb0 >= 0 ? op.rb0 : op.rb1;
                            const int cp = op.rb0 >= 0 ? op.pos1 : op.pos0;
                            with_rb<R>(rb, [&](auto B) { v = t_z<decltype(B)::value, NR>(x, y); });
                            if ((g_t >> cp) & 1) v = -v;
                        } else {
                            v = t_sum<NR>(x, y);
                            if (((g_t >> op.pos0) ^ (g_t >> op.pos1)) & 1) v = -v;
                        }
                        break;
                    default: break;
                }
                tap_store<RT>(v, stap, op.tap, nwarps, T);
            }
            break;
    }
}

// ---------------------------------------------------------------------------
// fused tile sweep
// ---------------------------------------------------------------------------
template <typename RT, int R, bool BWD>
__global__ void __launch_bounds__(512, 1) sweep_kernel(const SweepArgs a) {
    using V = typename CxT<RT>::T;
    constexpr int NR = 1 << R;
    constexpr int W = sizeof(RT) == 4 ? 4 : 3;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const DevSweep& sw = a.sw;
    const int k = sw.k;
    const uint32_t TS = 1u << k;
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    const int nwarps = (T + 31) >> 5;

    V* tile = reinterpret_cast<V*>(smem_raw);
    V* tile2 = tile + (BWD ? TS : 0);
    V* smat = tile2 + TS;
    double* stap = reinterpret_cast<double*>(smat + ((sw.n_mat + 1) & ~1));
    const int n_ops = sw.op_end - sw.op_begin;
    DevOp* sops = reinterpret_cast<DevOp*>(stap + ((sw.n_taps * nwarps + 1) & ~1));
    DevPhase* sph = reinterpret_cast<DevPhase*>(sops + n_ops);

    const uint32_t tile_id = blockIdx.x;
    const int b = blockIdx.y;
    const size_t N = size_t(1) << a.n;
    V* st = reinterpret_cast<V*>(a.psi) + (size_t)b * N;
    V* lm = BWD ? reinterpret_cast<V*>(a.lam) + (size_t)b * N : nullptr;

    uint32_t tile_base = 0;
    {
        uint32_t m = sw.out_mask, t = tile_id;
        while (m) {
            const uint32_t low = m & (0u - m);
            if (t & 1) tile_base |= low;
            t >>= 1;
            m ^= low;
        }
    }
    // memory offsets of the load/store loop index j (tile bits k-R .. k-1), in registers
    uint32_t jb[R];
#pragma unroll
    for (int r = 0; r < R; ++r) jb[r] = 1u << sw.tb[k - R + r];
    uint32_t g_ld = tile_base;
    for (int j = 0; j < k - R; ++j)
        if ((tid >> j) & 1) g_ld |= 1u << sw.tb[j];

    // HBM -> registers: every load in flight before the first shared-memory store
    V v0[NR];
    V v1[BWD ? NR : 1];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        uint32_t g = g_ld;
#pragma unroll
        for (int r = 0; r < R; ++r)
            if ((j >> r) & 1) g |= jb[r];
        if (!BWD && a.from_zero) {
            v0[j].x = (g == 0) ? RT(1) : RT(0);
            v0[j].y = RT(0);
        } else {
            v0[j] = st[g];
        }
        if constexpr (BWD) v1[j] = lm[g];
    }

    // op list, phases and gate matrices of this sweep -> shared memory
    for (int o = tid; o < n_ops; o += T) sops[o] = a.ops[sw.op_begin + o];
    for (int f = tid; f < sw.n_phases; f += T) sph[f] = a.phases[sw.phase_begin + f];
    {
        const V* gm = reinterpret_cast<const V*>(a.gmat) + (size_t)b * a.gmat_stride + a.gmat_pass_base + sw.mbase;
        for (int i = tid; i < sw.n_mat; i += T) smat[i] = gm[i];
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const uint32_t p = tid + (uint32_t)T * j;
        tile[swz<W>(p)] = v0[j];
        if constexpr (BWD) tile2[swz<W>(p)] = v1[j];
    }
    __syncthreads();

    for (int f = 0; f < sw.n_phases; ++f) {
        const DevPhase* ph = sph + f;
        uint32_t p_t = 0, g_t = tile_base;
        for (int j = 0; j < k - R; ++j) {
            const int tl = ph->thr_tl[j];
            if ((tid >> j) & 1) {
                p_t |= 1u << tl;
                g_t |= 1u << sw.tb[tl];
            }
        }
        uint32_t swr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) swr[r] = swz<W>(1u << ph->reg_tl[r]);
        const uint32_t s_t = swz<W>(p_t);
        V x[NR];
        V y[BWD ? NR : 1];
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            uint32_t si = s_t;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if ((i >> r) & 1) si ^= swr[r];
            x[i] = tile[si];
            if constexpr (BWD) y[i] = tile2[si];
        }
        uint32_t s_st = s_t;
        asm volatile("" : "+r"(s_st));
        const int ob = ph->op_begin - sw.op_begin, oe = ph->op_end - sw.op_begin;
        if (ob < oe) {
            DevOp nxt = sops[ob];
            for (int o = ob; o < oe; ++o) {
                const DevOp op = nxt;
                if (o + 1 < oe) nxt = sops[o + 1];  // prefetch: hides the shared-memory latency
                apply_op<RT, R, BWD>(op, x, y, g_t, smat, stap, nwarps, T);
            }
        }
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            uint32_t si = s_st;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if ((i >> r) & 1) si ^= swr[r];
            tile[si] = x[i];
            if constexpr (BWD) tile2[si] = y[i];
        }
        __syncthreads();
    }

    // shared tile -> registers -> HBM
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        const uint32_t p = tid + (uint32_t)T * j;
        v0[j] = tile[swz<W>(p)];
        if constexpr (BWD) v1[j] = tile2[swz<W>(p)];
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
        uint32_t g = g_ld;
#pragma unroll
        for (int r = 0; r < R; ++r)
            if ((j >> r) & 1) g |= jb[r];
        st[g] = v0[j];
        if constexpr (BWD) lm[g] = v1[j];
    }
    if constexpr (BWD) {
        const int tiles = gridDim.x;
        for (int t = tid; t < sw.n_taps; t += T) {
            double s = 0;
            for (int w = 0; w < nwarps; ++w) s += stap[t * nwarps + w];
            a.tap_part[((size_t)b * a.n_taps_total + sw.tap_begin + t) * tiles + tile_id] = s;
        }
    }
}


template <typename RT, int R, bool BWD>
cudaError_t launch_sweep_t(const SweepArgs& a, int batch, size_t smem, cudaStream_t s) {
    auto kern = sweep_kernel<RT, R, BWD>;
    static size_t configured = 0;  // per instantiation
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    dim3 grid(1u << (a.n - a.sw.k), batch);
    dim3 block(1u << (a.sw.k - R));
    kern<<<grid, block, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace qfb
