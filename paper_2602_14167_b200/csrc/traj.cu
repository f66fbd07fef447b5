// traj.cu -- projective measurements of batched trajectories (measure_collapse,
// reference circuit.cpp:391-429) for the trajectory workloads of SURVEY.md 8f
// row 4 (MIPT-Haar, experiments.cpp:210-250).  All reductions are fixed order.
#include "kernels.cuh"

namespace qfb {

namespace {

__device__ __forceinline__ uint32_t pdep32(uint32_t t, uint32_t m) {
    uint32_t r = 0;
    while (m) {
        const uint32_t low = m & (0u - m);
        if (t & 1) r |= low;
        t >>= 1;
        m ^= low;
    }
    return r;
}

// pdep32(t + k, m) from x = pdep32(t, m) and step = pdep32(k, m): the carry runs
// through the masked-out bits (no per-element bit loop)
__device__ __forceinline__ uint32_t pdep_add(uint32_t x, uint32_t step, uint32_t m) {
    return ((x | ~m) + step) & m;
}

// block (beta, b): sum of |psi[x]|^2 over x whose measured bits spell beta
template <typename V>
__global__ void __launch_bounds__(256) meas_hist_kernel(const V* psi, int n, const MeasRound* rounds, double* hist) {
    __shared__ double red[8];
    const int b = blockIdx.y;
    const uint32_t beta = blockIdx.x;
    const MeasRound r = rounds[b];
    if (r.count == 0 || beta >= (1u << r.count)) return;
    uint32_t mask = 0, dep = 0;
    for (int k = 0; k < r.count; ++k) {
        mask |= 1u << r.pos[k];
        if ((beta >> k) & 1) dep |= 1u << r.pos[k];
    }
    const uint32_t N = 1u << n, free = (N - 1) & ~mask;
    const uint32_t rest = 1u << (n - r.count);
    const V* ps = psi + (size_t)b * N;
    // walk the free bits as a counter: x -> ((x | mask) + step) & free, step = pdep(T)
    const uint32_t step = pdep32(blockDim.x, free);
    uint32_t x = pdep32(threadIdx.x, free);
    double acc = 0.0;
    for (uint32_t i = threadIdx.x; i < rest; i += blockDim.x) {
        const V a = ps[x | dep];
        acc += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
        x = ((x | mask) + step) & free;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        hist[(size_t)b * (1u << kMeasMax) + beta] = t;
    }
}

// thread per state: measure_collapse (d = 2) for each measurement in order
__global__ void meas_decide_kernel(const MeasRound* rounds, const double* hist, int batch, uint32_t* mask,
                                   uint32_t* bits, double* scale, int* outcomes) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const MeasRound r = rounds[b];
    const double* h = hist + (size_t)b * (1u << kMeasMax);
    uint32_t m = 0, o_bits = 0;
    double cum = 1.0, sc = 1.0;  // cum = product of the outcome probabilities so far
    for (int k = 0; k < r.count; ++k) {
        double a[2] = {0.0, 0.0};
        const uint32_t lowmask = (1u << k) - 1;
        for (uint32_t beta = 0; beta < (1u << r.count); ++beta)
            if ((beta & lowmask) == (o_bits & lowmask)) a[(beta >> k) & 1] += h[beta];
        const double probs[2] = {k ? a[0] / cum : a[0], k ? a[1] / cum : a[1]};
        int outcome = 1;
        double acc = 0.0;
        for (int o = 0; o < 2; ++o) {
            acc += probs[o];
            if (r.u[k] < acc) {
                outcome = o;
                break;
            }
        }
        const double p = probs[outcome];
        sc *= 1.0 / sqrt(p);
        cum *= p;
        o_bits |= (uint32_t)outcome << k;
        m |= 1u << r.pos[k];
        outcomes[(size_t)b * kMeasMax + k] = outcome;
    }
    uint32_t bb = 0;
    for (int k = 0; k < r.count; ++k)
        if ((o_bits >> k) & 1) bb |= 1u << r.pos[k];
    mask[b] = m;
    bits[b] = bb;
    scale[b] = sc;
}

template <typename V>
__global__ void meas_project_kernel(V* psi, int n, const MeasRound* rounds, const uint32_t* mask, const uint32_t* bits,
                                    const double* scale) {
    const int b = blockIdx.y;
    if (rounds[b].count == 0) return;
    const uint32_t N = 1u << n, m = mask[b], want = bits[b];
    const double sc = scale[b];
    V* ps = psi + (size_t)b * N;
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < N; x += gridDim.x * blockDim.x) {
        V a = ps[x];
        if ((x & m) == want) {
            a.x = (decltype(a.x))((double)a.x * sc);
            a.y = (decltype(a.y))((double)a.y * sc);
        } else {
            a.x = 0;
            a.y = 0;
        }
        ps[x] = a;
    }
}

template <typename V>
__global__ void set_basis0_kernel(V* psi, int n, int batch) {
    const uint32_t N = 1u << n;
    const size_t total = (size_t)batch * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        V a;
        a.x = (i % N) == 0 ? 1 : 0;
        a.y = 0;
        psi[i] = a;
    }
}

// inverse-CDF sampling (shadow_snapshots, shadows.cpp:64-78): chunk sums of |psi|^2
// in fixed order, then one thread per state walks the chunk sums and the hit
// chunk's amplitudes with a running sum as the reference does (acc += |a_i|^2,
// first i with u < acc; the last index when none)
template <typename V>
__global__ void __launch_bounds__(256) chunk_norms_kernel(const V* psi, int n, int chunk_bits, double* csum) {
    __shared__ double red[8];
    const int b = blockIdx.y;
    const size_t N = size_t(1) << n, C = size_t(1) << chunk_bits;
    const V* ps = psi + (size_t)b * N + (size_t)blockIdx.x * C;
    double acc = 0.0;
    for (size_t i = threadIdx.x; i < C; i += blockDim.x) {
        const V a = ps[i];
        acc += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        csum[(size_t)b * gridDim.x + blockIdx.x] = t;
    }
}

template <typename V>
__global__ void sample_pick_kernel(const V* psi, int n, int chunk_bits, const double* csum, const double* u, int batch,
                                   int64_t* hit) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const size_t N = size_t(1) << n, C = size_t(1) << chunk_bits, nc = N / C;
    const V* ps = psi + (size_t)b * N;
    const double* cs = csum + (size_t)b * nc;
    const double ub = u[b];
    double acc = 0.0;
    size_t c = 0;
    while (c < nc && !(ub < acc + cs[c])) acc += cs[c++];
    int64_t h = (int64_t)N - 1;
    for (size_t i = c * C; i < N; ++i) {
        const V a = ps[i];
        acc += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
        if (ub < acc) {
            h = (int64_t)i;
            break;
        }
    }
    hit[b] = h;
}

// Local operator on wires (w0[, w1]) of every state: amplitude quads / pairs in
// the local basis (w0 most significant), matrix shared (mstride = 0) or per state.
// Used by the noise trajectories for gates without channels and final Kraus branches.
template <typename V, int D>
__global__ void apply_local_kernel(V* psi, int n, int p0, int p1, const double2* m, int mstride) {
    const int b = blockIdx.y;
    const double2* mb = m + (size_t)b * mstride;
    double2 mm[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) mm[i] = mb[i];
    const uint32_t N = 1u << n, R = N / D;
    const uint32_t mask = D == 2 ? (1u << p0) : ((1u << p0) | (1u << p1));
    const uint32_t free = (N - 1) & ~mask;
    V* ps = psi + (size_t)b * N;
    const uint32_t stride = gridDim.x * blockDim.x, step = pdep32(stride, free);
    uint32_t base = pdep32(blockIdx.x * blockDim.x + threadIdx.x, free);
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride, base = pdep_add(base, step, free)) {
        uint32_t idx[D];
        double2 a[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            idx[i] = base | (D == 2 ? (i ? (1u << p0) : 0u)
                                    : (((i >> 1) & 1) ? (1u << p0) : 0u) | ((i & 1) ? (1u << p1) : 0u));
            const V v = ps[idx[i]];
            a[i] = make_double2((double)v.x, (double)v.y);
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double re = 0.0, im = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const double2 c = mm[i * D + j];
                re += c.x * a[j].x - c.y * a[j].y;
                im += c.x * a[j].y + c.y * a[j].x;
            }
            V o;
            o.x = (decltype(o.x))re;
            o.y = (decltype(o.y))im;
            ps[idx[i]] = o;
        }
    }
}

// Noise step pass: a D x D operator (the gate, shared, or a per-trajectory Kraus
// branch K/sqrt(p)) on wires (w0[, w1]) of every state, and the local density
// matrix of the RESULT on the same wires as fixed-order partials [b][part][D][D]
// (the next channel on that gate picks its branch from it).  One read + one write
// of the state replaces the separate operator and reduction passes.
template <typename V, int D>
__global__ void __launch_bounds__(256) apply_rho_kernel(V* psi, int n, int p0, int p1, const double2* m, int mstride,
                                                        double2* rho) {
    __shared__ double red[8][2 * D * D];
    const int b = blockIdx.y, part = blockIdx.x, parts = gridDim.x;
    const double2* mb = m + (size_t)b * mstride;
    double2 mm[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) mm[i] = mb[i];
    const uint32_t N = 1u << n, R = N / D;
    const uint32_t mask = D == 2 ? (1u << p0) : ((1u << p0) | (1u << p1));
    const uint32_t free = (N - 1) & ~mask;
    V* ps = psi + (size_t)b * N;
    double acc[2 * D * D];
#pragma unroll
    for (int i = 0; i < 2 * D * D; ++i) acc[i] = 0.0;
    const uint32_t r0 = (uint32_t)((uint64_t)R * part / parts), r1 = (uint32_t)((uint64_t)R * (part + 1) / parts);
    // two amplitude groups per iteration, both loaded before either is stored
    // (the stores would otherwise order every next load behind them)
    constexpr int U = 2;
    const uint32_t step1 = pdep32(blockDim.x, free), stepU = pdep32(U * blockDim.x, free);
    uint32_t base0 = pdep32(r0 + threadIdx.x, free);
    for (uint32_t r = r0 + threadIdx.x; r < r1; r += U * blockDim.x, base0 = pdep_add(base0, stepU, free)) {
        uint32_t idx[U][D];
        double2 a[U][D];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t ru = r + u * blockDim.x;
            live[u] = ru < r1;
            const uint32_t base = (u == 0 || !live[u]) ? base0 : pdep_add(base0, step1, free);
#pragma unroll
            for (int i = 0; i < D; ++i) {
                idx[u][i] = base | (D == 2 ? (i ? (1u << p0) : 0u)
                                           : (((i >> 1) & 1) ? (1u << p0) : 0u) | ((i & 1) ? (1u << p1) : 0u));
                const V v = ps[idx[u][i]];
                a[u][i] = make_double2((double)v.x, (double)v.y);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!live[u]) continue;
            double2 o[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double re = 0.0, im = 0.0;
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    const double2 c = mm[i * D + j];
                    re += c.x * a[u][j].x - c.y * a[u][j].y;
                    im += c.x * a[u][j].y + c.y * a[u][j].x;
                }
                V w;
                w.x = (decltype(w.x))re;
                w.y = (decltype(w.y))im;
                ps[idx[u][i]] = w;
                o[i] = make_double2((double)w.x, (double)w.y);  // the stored (rounded) amplitude
            }
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    acc[2 * (i * D + j)] += o[i].x * o[j].x + o[i].y * o[j].y;
                    acc[2 * (i * D + j) + 1] += o[i].y * o[j].x - o[i].x * o[j].y;
                }
        }
    }
#pragma unroll
    for (int i = 0; i < 2 * D * D; ++i) {
        double v = acc[i];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < 2 * D * D) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
        reinterpret_cast<double*>(rho + ((size_t)b * parts + part) * D * D)[threadIdx.x] = t;
    }
}

// Noise step with the previous channel's branch folded in: the pending
// per-trajectory K/sqrt(p) on wires Wp, then the gate on the disjoint wires Wj,
// then the local rho partials on Wj -- one state pass instead of two.  Local
// amplitude index l = (ip << log2 DJ) | ij (wires[0] most significant in each).
template <typename V, int DP, int DJ>
__global__ void __launch_bounds__(256) apply2_rho_kernel(V* psi, int n, int q0, int q1, const double2* kp, int p0,
                                                         int p1, const double2* g, double2* rho) {
    __shared__ double red[8][2 * DJ * DJ];
    const int b = blockIdx.y, part = blockIdx.x, parts = gridDim.x;
    const double2* kb = kp + (size_t)b * DP * DP;
    double2 km[DP * DP], gm[DJ * DJ];
#pragma unroll
    for (int i = 0; i < DP * DP; ++i) km[i] = kb[i];
#pragma unroll
    for (int i = 0; i < DJ * DJ; ++i) gm[i] = g[i];
    const uint32_t N = 1u << n, R = N / (DP * DJ);
    const uint32_t mp = DP == 2 ? (1u << q0) : ((1u << q0) | (1u << q1));
    const uint32_t mj = DJ == 2 ? (1u << p0) : ((1u << p0) | (1u << p1));
    const uint32_t free = (N - 1) & ~(mp | mj);
    V* ps = psi + (size_t)b * N;
    double acc[2 * DJ * DJ];
#pragma unroll
    for (int i = 0; i < 2 * DJ * DJ; ++i) acc[i] = 0.0;
    auto dep = [](int i, int D, int w0, int w1) -> uint32_t {
        return D == 2 ? (i ? (1u << w0) : 0u) : ((((i >> 1) & 1) ? (1u << w0) : 0u) | ((i & 1) ? (1u << w1) : 0u));
    };
    const uint32_t r0 = (uint32_t)((uint64_t)R * part / parts), r1 = (uint32_t)((uint64_t)R * (part + 1) / parts);
    const uint32_t step = pdep32(blockDim.x, free);
    uint32_t base = pdep32(r0 + threadIdx.x, free);
    for (uint32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x, base = pdep_add(base, step, free)) {
        uint32_t idx[DP * DJ];
        double2 a[DP * DJ];
#pragma unroll
        for (int ip = 0; ip < DP; ++ip)
#pragma unroll
            for (int ij = 0; ij < DJ; ++ij) {
                const int l = ip * DJ + ij;
                idx[l] = base | dep(ip, DP, q0, q1) | dep(ij, DJ, p0, p1);
                const V v = ps[idx[l]];
                a[l] = make_double2((double)v.x, (double)v.y);
            }
        // pending Kraus branch on Wp (same arithmetic as apply_local_kernel)
#pragma unroll
        for (int ij = 0; ij < DJ; ++ij) {
            double2 t[DP];
#pragma unroll
            for (int i = 0; i < DP; ++i) {
                double re = 0.0, im = 0.0;
#pragma unroll
                for (int j = 0; j < DP; ++j) {
                    const double2 c = km[i * DP + j], x = a[j * DJ + ij];
                    re += c.x * x.x - c.y * x.y;
                    im += c.x * x.y + c.y * x.x;
                }
                t[i] = make_double2(re, im);
            }
#pragma unroll
            for (int i = 0; i < DP; ++i) {  // round to the state precision, as a separate pass would store
                V w;
                w.x = (decltype(w.x))t[i].x;
                w.y = (decltype(w.y))t[i].y;
                a[i * DJ + ij] = make_double2((double)w.x, (double)w.y);
            }
        }
        // gate on Wj, store, rho partials of the result
#pragma unroll
        for (int ip = 0; ip < DP; ++ip) {
            double2 o[DJ];
#pragma unroll
            for (int i = 0; i < DJ; ++i) {
                double re = 0.0, im = 0.0;
#pragma unroll
                for (int j = 0; j < DJ; ++j) {
                    const double2 c = gm[i * DJ + j], x = a[ip * DJ + j];
                    re += c.x * x.x - c.y * x.y;
                    im += c.x * x.y + c.y * x.x;
                }
                V w;
                w.x = (decltype(w.x))re;
                w.y = (decltype(w.y))im;
                ps[idx[ip * DJ + i]] = w;
                o[i] = make_double2((double)w.x, (double)w.y);
            }
#pragma unroll
            for (int i = 0; i < DJ; ++i)
#pragma unroll
                for (int j = 0; j < DJ; ++j) {
                    acc[2 * (i * DJ + j)] += o[i].x * o[j].x + o[i].y * o[j].y;
                    acc[2 * (i * DJ + j) + 1] += o[i].y * o[j].x - o[i].x * o[j].y;
                }
        }
    }
#pragma unroll
    for (int i = 0; i < 2 * DJ * DJ; ++i) {
        double v = acc[i];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < 2 * DJ * DJ) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
        reinterpret_cast<double*>(rho + ((size_t)b * parts + part) * DJ * DJ)[threadIdx.x] = t;
    }
}

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// branch probability p_k = tr(K_k rho K_k^dagger) (reference noise.cpp:178-185)
__device__ double kraus_prob(const double* K, const double2* r, int D) {
    double pk = 0.0;
    for (int a = 0; a < D; ++a) {
        double2 sa = make_double2(0.0, 0.0);
        for (int i = 0; i < D; ++i) {
            const double2 ki = make_double2(K[(a * 4 + i) * 2], K[(a * 4 + i) * 2 + 1]);
            for (int j = 0; j < D; ++j) {
                const double2 kj = make_double2(K[(a * 4 + j) * 2], -K[(a * 4 + j) * 2 + 1]);
                const double2 t = zmul(zmul(ki, r[i * D + j]), kj);
                sa.x += t.x;
                sa.y += t.y;
            }
        }
        pk += sa.x;
    }
    return pk;
}

// One warp per trajectory: the reference's branch pick for one channel
// application (noise.cpp:186-195: first k with u * sum(p) < running sum, else the
// last), from the rho partials (lane l sums parts l, l + 32, ... in order, then a
// fixed xor-shuffle tree: the order depends only on n); writes K_pick / sqrt(p_pick)
// and accumulates log p.  err = 1 when every branch probability vanishes.
__global__ void __launch_bounds__(128) kraus_pick_kernel(const double2* rho, int parts, int D, const double* kraus,
                                                         int k0, int k1, const double* u, int u_stride, int app,
                                                         double2* kout, double* logp, int* err, int batch) {
    const int b = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (b >= batch) return;
    double2 r[16];
    for (int e = 0; e < 16; ++e) r[e] = make_double2(0.0, 0.0);
    for (int pt = lane; pt < parts; pt += 32)
        for (int e = 0; e < D * D; ++e) {
            const double2 v = rho[((size_t)b * parts + pt) * D * D + e];
            r[e].x += v.x;
            r[e].y += v.y;
        }
    for (int e = 0; e < D * D; ++e)
        for (int o = 16; o > 0; o >>= 1) {
            r[e].x += __shfl_xor_sync(0xffffffffu, r[e].x, o);
            r[e].y += __shfl_xor_sync(0xffffffffu, r[e].y, o);
        }
    if (lane) return;
    double acc = 0.0;
    for (int k = k0; k < k1; ++k) acc += kraus_prob(kraus + 32 * (size_t)k, r, D);
    if (!(acc > 1e-14)) {
        atomicExch(err, 1);
        for (int e = 0; e < D * D; ++e) kout[(size_t)b * D * D + e] = make_double2(0.0, 0.0);
        return;
    }
    const double uu = u[(size_t)b * u_stride + app] * acc;
    int pick = k1 - 1;
    double pp = 0.0, run = 0.0;
    bool hit = false;
    for (int k = k0; k < k1; ++k) {
        const double pk = kraus_prob(kraus + 32 * (size_t)k, r, D);
        run += pk;
        pp = pk;
        if (uu < run) {
            pick = k;
            hit = true;
            break;
        }
    }
    if (!hit) pp = kraus_prob(kraus + 32 * (size_t)pick, r, D);
    const double sc = 1.0 / sqrt(pp);
    const double* K = kraus + 32 * (size_t)pick;
    for (int a = 0; a < D; ++a)
        for (int i = 0; i < D; ++i)
            kout[(size_t)b * D * D + a * D + i] = make_double2(K[(a * 4 + i) * 2] * sc, K[(a * 4 + i) * 2 + 1] * sc);
    logp[b] += log(pp / acc) + log(acc);
}

// Generic k-wire operator on one complex128 state (apply_local_unitary,
// reference circuit.cpp:147-175: wires[0] most significant local bit).
// Small k: a thread per amplitude group, the 2^K amplitudes in registers, U in
// shared memory.  pos[i] = memory bit position of wires[i].
template <int K>
__global__ void __launch_bounds__(256) apply_unitary_small_kernel(double2* psi, int n, const int* pos_g,
                                                                  const double2* u) {
    constexpr int DK = 1 << K;
    __shared__ double2 su[DK * DK];
    __shared__ int pos[K];
    for (int i = threadIdx.x; i < DK * DK; i += blockDim.x) su[i] = u[i];
    if (threadIdx.x < K) pos[threadIdx.x] = pos_g[threadIdx.x];
    __syncthreads();
    uint32_t mask = 0;
    for (int i = 0; i < K; ++i) mask |= 1u << pos[i];
    const uint32_t N = 1u << n, free = (N - 1) & ~mask, G = N >> K;
    uint32_t off[DK];
#pragma unroll
    for (int j = 0; j < DK; ++j) {
        uint32_t o = 0;
        for (int i = 0; i < K; ++i)
            if ((j >> (K - 1 - i)) & 1) o |= 1u << pos[i];
        off[j] = o;
    }
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
        const uint32_t base = pdep32(g, free);
        double2 a[DK];
#pragma unroll
        for (int j = 0; j < DK; ++j) a[j] = psi[base | off[j]];
#pragma unroll
        for (int i = 0; i < DK; ++i) {
            double re = 0.0, im = 0.0;
#pragma unroll
            for (int j = 0; j < DK; ++j) {
                const double2 c = su[i * DK + j];
                re += c.x * a[j].x - c.y * a[j].y;
                im += c.x * a[j].y + c.y * a[j].x;
            }
            psi[base | off[i]] = make_double2(re, im);
        }
    }
}

// Large k: a CTA per amplitude group, the group in shared memory, thread i ->
// output rows i, i + T, ...; U column-major (ut[j * DK + i] = U[i][j]) so a
// column read is coalesced across the rows.
__global__ void __launch_bounds__(256) apply_unitary_large_kernel(double2* psi, int n, int k, const int* pos_g,
                                                                  const double2* ut) {
    extern __shared__ double2 grp[];
    const uint32_t DK = 1u << k, N = 1u << n;
    uint32_t mask = 0;
    for (int i = 0; i < k; ++i) mask |= 1u << pos_g[i];
    const uint32_t free = (N - 1) & ~mask, G = N >> k;
    auto offset = [&](uint32_t j) {
        uint32_t o = 0;
        for (int i = 0; i < k; ++i)
            if ((j >> (k - 1 - i)) & 1) o |= 1u << pos_g[i];
        return o;
    };
    for (uint32_t g = blockIdx.x; g < G; g += gridDim.x) {
        const uint32_t base = pdep32(g, free);
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < DK; j += blockDim.x) grp[j] = psi[base | offset(j)];
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < DK; i += blockDim.x) {
            double re = 0.0, im = 0.0;
            for (uint32_t j = 0; j < DK; ++j) {
                const double2 c = ut[(size_t)j * DK + i], x = grp[j];
                re += c.x * x.x - c.y * x.y;
                im += c.x * x.y + c.y * x.x;
            }
            psi[base | offset(i)] = make_double2(re, im);
        }
    }
}

}  // namespace

cudaError_t launch_apply_unitary(double2* psi, int n, int k, const int* d_pos, const double2* d_u, const double2* d_ut,
                                 cudaStream_t s) {
    const uint32_t G = (1u << n) >> k;
    const unsigned grid_small = std::max(1u, std::min<uint32_t>((G + 255) / 256, 2048));
    switch (k) {
        case 1: apply_unitary_small_kernel<1><<<grid_small, 256, 0, s>>>(psi, n, d_pos, d_u); break;
        case 2: apply_unitary_small_kernel<2><<<grid_small, 256, 0, s>>>(psi, n, d_pos, d_u); break;
        case 3: apply_unitary_small_kernel<3><<<grid_small, 256, 0, s>>>(psi, n, d_pos, d_u); break;
        case 4: apply_unitary_small_kernel<4><<<grid_small, 256, 0, s>>>(psi, n, d_pos, d_u); break;
        default: {
            const size_t sm = ((size_t)1 << k) * sizeof(double2);
            cudaError_t e = cudaFuncSetAttribute(apply_unitary_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)sm);
            if (e != cudaSuccess) return e;
            apply_unitary_large_kernel<<<std::max(1u, std::min<uint32_t>(G, 4096)), 256, sm, s>>>(psi, n, k, d_pos, d_ut);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_apply_rho(int prec, void* psi, int n, int batch, int p0, int p1, const double2* m, bool per_state,
                             double2* rho, cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    const int D = p1 >= 0 ? 4 : 2;
    const dim3 grid(local_rho_parts(n), batch);
    const int ms = per_state ? D * D : 0;
    if (prec == 1) {
        if (D == 2) apply_rho_kernel<double2, 2><<<grid, 256, 0, s>>>((double2*)psi, n, p0, p1, m, ms, rho);
        else apply_rho_kernel<double2, 4><<<grid, 256, 0, s>>>((double2*)psi, n, p0, p1, m, ms, rho);
    } else {
        if (D == 2) apply_rho_kernel<float2, 2><<<grid, 256, 0, s>>>((float2*)psi, n, p0, p1, m, ms, rho);
        else apply_rho_kernel<float2, 4><<<grid, 256, 0, s>>>((float2*)psi, n, p0, p1, m, ms, rho);
    }
    return cudaGetLastError();
}

cudaError_t launch_apply2_rho(int prec, void* psi, int n, int batch, int q0, int q1, const double2* kp, int p0,
                              int p1, const double2* g, double2* rho, cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    const int DP = q1 >= 0 ? 4 : 2, DJ = p1 >= 0 ? 4 : 2;
    const dim3 grid(local_rho_parts(n), batch);
#define QF_A2(T, A, B) apply2_rho_kernel<T, A, B><<<grid, 256, 0, s>>>((T*)psi, n, q0, q1, kp, p0, p1, g, rho)
    if (prec == 1) {
        if (DP == 2 && DJ == 2) QF_A2(double2, 2, 2);
        else if (DP == 2) QF_A2(double2, 2, 4);
        else if (DJ == 2) QF_A2(double2, 4, 2);
        else QF_A2(double2, 4, 4);
    } else {
        if (DP == 2 && DJ == 2) QF_A2(float2, 2, 2);
        else if (DP == 2) QF_A2(float2, 2, 4);
        else if (DJ == 2) QF_A2(float2, 4, 2);
        else QF_A2(float2, 4, 4);
    }
#undef QF_A2
    return cudaGetLastError();
}

cudaError_t launch_kraus_pick(const double2* rho, int parts, int D, const double* kraus, int k0, int k1, const double* u,
                              int u_stride, int app, double2* kout, double* logp, int* err, int batch, cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    kraus_pick_kernel<<<(batch + 3) / 4, 128, 0, s>>>(rho, parts, D, kraus, k0, k1, u, u_stride, app, kout, logp,
                                                          err, batch);
    return cudaGetLastError();
}

cudaError_t launch_apply_local(int prec, void* psi, int n, int batch, int p0, int p1, const double2* m, bool per_state,
                               cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    const int D = p1 >= 0 ? 4 : 2;
    const uint32_t R = (1u << n) / D;
    dim3 grid(std::max(1u, std::min<uint32_t>((R + 255) / 256, 512)), batch);
    const int ms = per_state ? D * D : 0;
    if (prec == 1) {
        if (D == 2) apply_local_kernel<double2, 2><<<grid, 256, 0, s>>>((double2*)psi, n, p0, p1, m, ms);
        else apply_local_kernel<double2, 4><<<grid, 256, 0, s>>>((double2*)psi, n, p0, p1, m, ms);
    } else {
        if (D == 2) apply_local_kernel<float2, 2><<<grid, 256, 0, s>>>((float2*)psi, n, p0, p1, m, ms);
        else apply_local_kernel<float2, 4><<<grid, 256, 0, s>>>((float2*)psi, n, p0, p1, m, ms);
    }
    return cudaGetLastError();
}

// fixed number of rho partials per state (one CTA each): ~2^(n-9) amplitudes per CTA
int local_rho_parts(int n) { return n < 10 ? 1 : 1 << std::min(8, n - 10); }

int sample_chunk_bits(int n) { return n > 10 ? 10 : n; }

cudaError_t launch_sample(int prec, const void* psi, int n, int batch, const double* u, double* csum, int64_t* hit,
                          cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    const int cb = sample_chunk_bits(n);
    dim3 grid(1u << (n - cb), batch);
    if (prec == 1) {
        chunk_norms_kernel<double2><<<grid, 256, 0, s>>>((const double2*)psi, n, cb, csum);
        sample_pick_kernel<double2><<<(batch + 127) / 128, 128, 0, s>>>((const double2*)psi, n, cb, csum, u, batch, hit);
    } else {
        chunk_norms_kernel<float2><<<grid, 256, 0, s>>>((const float2*)psi, n, cb, csum);
        sample_pick_kernel<float2><<<(batch + 127) / 128, 128, 0, s>>>((const float2*)psi, n, cb, csum, u, batch, hit);
    }
    return cudaGetLastError();
}

cudaError_t launch_meas_hist(int prec, const void* psi, int n, int batch, const MeasRound* rounds, int max_count,
                             double* hist, cudaStream_t s) {
    if (batch == 0 || max_count == 0) return cudaSuccess;
    dim3 grid(1u << max_count, batch);
    if (prec == 1)
        meas_hist_kernel<double2><<<grid, 256, 0, s>>>((const double2*)psi, n, rounds, hist);
    else
        meas_hist_kernel<float2><<<grid, 256, 0, s>>>((const float2*)psi, n, rounds, hist);
    return cudaGetLastError();
}

cudaError_t launch_meas_decide(const MeasRound* rounds, const double* hist, int batch, uint32_t* mask, uint32_t* bits,
                               double* scale, int* outcomes, cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    meas_decide_kernel<<<(batch + 127) / 128, 128, 0, s>>>(rounds, hist, batch, mask, bits, scale, outcomes);
    return cudaGetLastError();
}

cudaError_t launch_meas_project(int prec, void* psi, int n, int batch, const MeasRound* rounds, const uint32_t* mask,
                                const uint32_t* bits, const double* scale, cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    const uint32_t N = 1u << n;
    dim3 grid(std::max(1u, std::min<uint32_t>(N / 1024, 256)), batch);
    if (prec == 1)
        meas_project_kernel<double2><<<grid, 256, 0, s>>>((double2*)psi, n, rounds, mask, bits, scale);
    else
        meas_project_kernel<float2><<<grid, 256, 0, s>>>((float2*)psi, n, rounds, mask, bits, scale);
    return cudaGetLastError();
}

cudaError_t launch_set_basis0(int prec, void* psi, int n, int batch, cudaStream_t s) {
    if (batch == 0) return cudaSuccess;
    if (prec == 1)
        set_basis0_kernel<double2><<<148 * 8, 256, 0, s>>>((double2*)psi, n, batch);
    else
        set_basis0_kernel<float2><<<148 * 8, 256, 0, s>>>((float2*)psi, n, batch);
    return cudaGetLastError();
}

}  // namespace qfb
