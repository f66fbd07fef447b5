// eig.cu -- batched Hermitian eigenvalues for the MIPT half-chain entropy
// (reference circuit.cpp:431-470, subsystem_entropy: JacobiSVD of psi reshaped to
// dk x de, entropy of the squared singular values).  The squared singular values
// are the eigenvalues of rho = A^H A (dk x dk, built by a batched ZGEMM); here:
//
//  1. hetrd_kernel: Householder reduction of every rho to a real symmetric
//     tridiagonal (the LAPACK zhetd2 / zlarfg recurrences, lower form), one CTA per
//     matrix.  Full column-major storage (both triangles updated) so every matrix
//     sweep is coalesced: thread r owns rows r, r + T, ... and walks the columns.
//     Step k updates the trailing block's first column (A22 -= v w^H + w v^H),
//     derives the next reflector from it, then sweeps the rest of the block once:
//     the rank-2 update and the next step's p = tau' A33 v' in the same pass, so
//     every step is one read + one write of the trailing block (2 L^2 complex
//     moves; (2/3) m^3 over the reduction).
//  2. tridiag_bisect_kernel: all eigenvalues of (d, e) by Sturm-count bisection
//     (LAPACK dstebz-style pivot guard), one thread per eigenvalue, ascending.
//
// Everything is double precision for both state precisions (a complex64 spectrum
// loses the small Schmidt values) and every reduction is fixed order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace qfb {

namespace {

__device__ __forceinline__ double2 zmul_(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zconjmul_(double2 a, double2 b) {  // conj(a) * b
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// fixed-order CTA sum (warp xor tree, then the warps in order); all threads get it
template <int NV>
__device__ void block_sum(double (&x)[NV], double (*red)[NV]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int c = 0; c < NV; ++c)
        for (int o = 16; o > 0; o >>= 1) x[c] += __shfl_xor_sync(0xffffffffu, x[c], o);
    __syncthreads();  // red[] reuse
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < NV; ++c) red[wid][c] = x[c];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += red[w][c];
        x[c] = t;
    }
}

// RPT rows per thread (m <= RPT * blockDim.x).  smem: v (reflector of this step),
// w (its rank-2 partner), vn (next reflector), p (tau A22 v of this step).
template <int RPT, int UN>
__global__ void __launch_bounds__(1024, 1) hetrd_kernel(double2* A, int m, double* d_out, double* e_out) {
    extern __shared__ __align__(16) double2 hsm[];
    __shared__ double red[32][2];
    double2* v = hsm;
    double2* w = hsm + m;
    double2* vn = hsm + 2 * m;
    double2* p = hsm + 3 * m;
    const int T = blockDim.x, tid = threadIdx.x;
    double2* Ab = A + (size_t)blockIdx.x * m * m;
    double* d = d_out + (size_t)blockIdx.x * m;
    double* e = e_out + (size_t)blockIdx.x * m;

    // Reflector of column k of the current matrix, A[k+1 .., k] (zlarfg): writes
    // vr[0 .. L) (vr[0] = 1), d[k], e[k] = beta; returns tau (0: identity).
    auto reflector = [&](int k, double2* vr) {
        const int L = m - k - 1;
        const double2* col = Ab + (size_t)k * m + (k + 1);
        double s[1] = {0.0};
        for (int i = tid + 1; i < L; i += T) {
            const double2 x = col[i];
            s[0] += x.x * x.x + x.y * x.y;
        }
        block_sum<1>(s, reinterpret_cast<double(*)[1]>(red));
        const double2 alpha = col[0];
        double beta;
        double2 tau;
        if (s[0] == 0.0 && alpha.y == 0.0) {
            tau = make_double2(0.0, 0.0);
            beta = alpha.x;
        } else {
            beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + s[0]), alpha.x);
            tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
            const double2 den = make_double2(alpha.x - beta, alpha.y);  // scal = 1 / (alpha - beta)
            const double dd = den.x * den.x + den.y * den.y;
            const double2 scal = make_double2(den.x / dd, -den.y / dd);
            for (int i = tid; i < L; i += T) vr[i] = i == 0 ? make_double2(1.0, 0.0) : zmul_(col[i], scal);
        }
        if (tid == 0) {
            d[k] = Ab[(size_t)k * m + k].x;
            e[k] = beta;
        }
        __syncthreads();
        return tau;
    };
    // p = tau * A22 v on its own (first step, and after an identity reflector)
    auto matvec = [&](int k, double2 tau) {
        const int L = m - k - 1;
        const double2* A22 = Ab + (size_t)(k + 1) * m + (k + 1);
        double2 acc[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) acc[q] = make_double2(0.0, 0.0);
        for (int j = 0; j < L; ++j) {
            const double2 vj = v[j];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int r = tid + q * T;
                if (r < L) {
                    const double2 t = zmul_(A22[(size_t)j * m + r], vj);
                    acc[q].x += t.x;
                    acc[q].y += t.y;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q)
            if (tid + q * T < L) p[tid + q * T] = zmul_(tau, acc[q]);
        __syncthreads();
    };

    if (m == 1) {
        if (tid == 0) d[0] = Ab[0].x;
        return;
    }
    double2 tau = reflector(0, v);
    if (tau.x != 0.0 || tau.y != 0.0) matvec(0, tau);
    for (int k = 0; k + 1 < m; ++k) {
        const int L = m - k - 1;  // trailing block A22 = A[k+1 .., k+1 ..], L x L
        double2* A22 = Ab + (size_t)(k + 1) * m + (k + 1);
        const bool last = k + 2 >= m;
        if (tau.x == 0.0 && tau.y == 0.0) {  // identity reflector: nothing to update
            if (last) {
                if (tid == 0) d[k + 1] = A22[0].x;
            } else {
                tau = reflector(k + 1, v);
                if (tau.x != 0.0 || tau.y != 0.0) matvec(k + 1, tau);
            }
            continue;
        }
        // w = p - (tau / 2) (p^H v) v
        double dot[2] = {0.0, 0.0};
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * T;
            if (r < L) {
                const double2 t = zconjmul_(p[r], v[r]);
                dot[0] += t.x;
                dot[1] += t.y;
            }
        }
        block_sum<2>(dot, red);
        const double2 a2 = zmul_(make_double2(-0.5 * tau.x, -0.5 * tau.y), make_double2(dot[0], dot[1]));
        double2 vr[RPT], wr[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * T;
            if (r < L) {
                vr[q] = v[r];
                const double2 t = zmul_(a2, vr[q]);
                wr[q] = make_double2(p[r].x + t.x, p[r].y + t.y);
                w[r] = wr[q];
            }
        }
        __syncthreads();
        // column 0 of the update first (it is the next step's reflector column)
        {
            const double2 w0 = w[0], v0 = v[0];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int r = tid + q * T;
                if (r < L) {
                    const double2 a = A22[r];
                    const double2 t1 = zmul_(vr[q], make_double2(w0.x, -w0.y));
                    const double2 t2 = zmul_(wr[q], make_double2(v0.x, -v0.y));
                    A22[r] = make_double2(a.x - t1.x - t2.x, a.y - t1.y - t2.y);
                }
            }
        }
        __syncthreads();
        if (last) {
            if (tid == 0) d[k + 1] = A22[0].x;
            break;
        }
        const double2 tn = reflector(k + 1, vn);
        const bool nxt = tn.x != 0.0 || tn.y != 0.0;
        // rest of the rank-2 update A22 -= v w^H + w v^H, column by column (coalesced),
        // fused with the next step's p = tn * A33 vn (A33 = A22[1 .., 1 ..])
        double2 acc[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) acc[q] = make_double2(0.0, 0.0);
        int j = 1;
        for (; j + UN <= L; j += UN) {
            double2 a[RPT][UN];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int r = tid + q * T;
                if (r < L)
#pragma unroll
                    for (int u = 0; u < UN; ++u) a[q][u] = A22[(size_t)(j + u) * m + r];
            }
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                const double2 wj = w[j + u], vj = v[j + u], vnj = nxt ? vn[j + u - 1] : make_double2(0.0, 0.0);
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const int r = tid + q * T;
                    if (r < L) {
                        const double2 t1 = zmul_(vr[q], make_double2(wj.x, -wj.y));
                        const double2 t2 = zmul_(wr[q], make_double2(vj.x, -vj.y));
                        const double2 nv = make_double2(a[q][u].x - t1.x - t2.x, a[q][u].y - t1.y - t2.y);
                        A22[(size_t)(j + u) * m + r] = nv;
                        const double2 t = zmul_(nv, vnj);
                        acc[q].x += t.x;
                        acc[q].y += t.y;
                    }
                }
            }
        }
        for (; j < L; ++j) {
            const double2 wj = w[j], vj = v[j], vnj = nxt ? vn[j - 1] : make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int r = tid + q * T;
                if (r < L) {
                    const double2 a = A22[(size_t)j * m + r];
                    const double2 t1 = zmul_(vr[q], make_double2(wj.x, -wj.y));
                    const double2 t2 = zmul_(wr[q], make_double2(vj.x, -vj.y));
                    const double2 nv = make_double2(a.x - t1.x - t2.x, a.y - t1.y - t2.y);
                    A22[(size_t)j * m + r] = nv;
                    const double2 t = zmul_(nv, vnj);
                    acc[q].x += t.x;
                    acc[q].y += t.y;
                }
            }
        }
        __syncthreads();  // every read of p, v, w of this step is done
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * T;
            if (r >= 1 && r < L) p[r - 1] = zmul_(tn, acc[q]);  // row r of A22 = row r - 1 of A33
        }
        for (int i = tid; i < L - 1; i += T) v[i] = vn[i];
        tau = tn;
        __syncthreads();
    }
}

// Eigenvalues (ascending) of the real symmetric tridiagonal (d[0 .. m), e[0 .. m-1))
// by bisection on the Sturm count, thread j -> the j-th smallest.
__global__ void __launch_bounds__(1024) tridiag_bisect_kernel(const double* d_in, const double* e_in, int m,
                                                              double* w_out) {
    extern __shared__ double tsm[];
    double* d = tsm;
    double* e2 = tsm + m;
    __shared__ double red[32][2];
    const int T = blockDim.x, tid = threadIdx.x;
    const double* db = d_in + (size_t)blockIdx.x * m;
    const double* eb = e_in + (size_t)blockIdx.x * m;
    double lo_hi[2] = {1e300, -1e300};
    double emax2[1] = {0.0};
    for (int i = tid; i < m; i += T) {
        d[i] = db[i];
        const double el = i > 0 ? fabs(eb[i - 1]) : 0.0, er = i + 1 < m ? fabs(eb[i]) : 0.0;
        e2[i] = i + 1 < m ? eb[i] * eb[i] : 0.0;
        emax2[0] = fmax(emax2[0], e2[i]);
        lo_hi[0] = fmin(lo_hi[0], d[i] - el - er);
        lo_hi[1] = fmax(lo_hi[1], d[i] + el + er);
    }
    // (min / max reductions: order-independent)
    for (int o = 16; o > 0; o >>= 1) {
        lo_hi[0] = fmin(lo_hi[0], __shfl_xor_sync(0xffffffffu, lo_hi[0], o));
        lo_hi[1] = fmax(lo_hi[1], __shfl_xor_sync(0xffffffffu, lo_hi[1], o));
        emax2[0] = fmax(emax2[0], __shfl_xor_sync(0xffffffffu, emax2[0], o));
    }
    __shared__ double em[32];
    if ((tid & 31) == 0) {
        red[tid >> 5][0] = lo_hi[0];
        red[tid >> 5][1] = lo_hi[1];
        em[tid >> 5] = emax2[0];
    }
    __syncthreads();
    double gl = 1e300, gu = -1e300, e2m = 0.0;
    for (int wq = 0; wq < (T >> 5); ++wq) {
        gl = fmin(gl, red[wq][0]);
        gu = fmax(gu, red[wq][1]);
        e2m = fmax(e2m, em[wq]);
    }
    const double safmin = 2.2250738585072014e-308;
    const double pivmin = safmin * fmax(1.0, e2m);
    const double bnorm = fmax(fabs(gl), fabs(gu));
    gl -= 2.0 * 2.220446049250313e-16 * bnorm * m + 2.0 * pivmin;
    gu += 2.0 * 2.220446049250313e-16 * bnorm * m + 2.0 * pivmin;
    auto count_below = [&](double x) {  // number of eigenvalues < x
        int c = 0;
        double q = d[0] - x;
        if (fabs(q) < pivmin) q = -pivmin;
        c += q < 0.0;
        for (int i = 1; i < m; ++i) {
            q = d[i] - x - e2[i - 1] / q;
            if (fabs(q) < pivmin) q = -pivmin;
            c += q < 0.0;
        }
        return c;
    };
    for (int j = tid; j < m; j += T) {
        double lo = gl, hi = gu;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (mid <= lo || mid >= hi) break;  // interval at double resolution
            if (hi - lo <= 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)) + pivmin) break;
            if (count_below(mid) > j) hi = mid;
            else lo = mid;
        }
        w_out[(size_t)blockIdx.x * m + j] = 0.5 * (lo + hi);
    }
}

}  // namespace

cudaError_t launch_hermitian_eigvals(double2* A, int m, int batch, double* d, double* e, double* w, cudaStream_t s) {
    if (batch == 0 || m == 0) return cudaSuccess;
    const int T = std::min(1024, ((m + 31) / 32) * 32);
    const int rpt = (m + T - 1) / T;
    const size_t hs = 4 * (size_t)m * sizeof(double2);
    cudaError_t err = cudaSuccess;
    static const int un = [] {  // columns in flight per thread in the fused sweep (development A/B)
        const char* e = std::getenv("QF_HETRD_UNROLL");
        return e && std::atoi(e) == 8 ? 8 : e && std::atoi(e) == 2 ? 2 : 4;
    }();
#define QF_HT(R_, U_)                                                                                     \
    do {                                                                                                  \
        err = cudaFuncSetAttribute(hetrd_kernel<R_, U_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs); \
        if (err == cudaSuccess) hetrd_kernel<R_, U_><<<batch, T, hs, s>>>(A, m, d, e);                     \
    } while (0)
    if (rpt <= 1) {
        if (un == 8) QF_HT(1, 8);
        else if (un == 2) QF_HT(1, 2);
        else QF_HT(1, 4);
    } else if (rpt <= 2) {
        if (un == 8) QF_HT(2, 8);
        else if (un == 2) QF_HT(2, 2);
        else QF_HT(2, 4);
    } else {
        return cudaErrorInvalidValue;  // m > 2048 (v, w, v', p staged in shared memory)
    }
#undef QF_HT
    if (err != cudaSuccess) return err;
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    const size_t bs = 2 * (size_t)m * sizeof(double);
    err = cudaFuncSetAttribute(tridiag_bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bs);
    if (err != cudaSuccess) return err;
    tridiag_bisect_kernel<<<batch, T, bs, s>>>(d, e, m, w);
    return cudaGetLastError();
}

}  // namespace qfb
