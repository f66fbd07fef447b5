// coo.cu -- pauli_sum_to_coo on the GPU (reference src/pauli.cpp:89-153,
// SURVEY.md 8f row 3; the construction the paper times in Table I).
//
// Row r of H = sum_t w_t P_t has one entry per distinct flip mask f: column
// r ^ f with value sum_{t: f_t = f} w_t i^{y_t} (-1)^{popc((r ^ f) & z_t)}
// (term_value, pauli.cpp:79-85).  Exact zeros are dropped and columns are
// ascending within a row, so the output is the reference's canonical form.
// Pass 1 counts per row, a cub scan gives offsets, pass 2 writes.
#include <cub/device/device_scan.cuh>

#include "kernels.cuh"

namespace qfb {

namespace {

constexpr int kThreadRowMax = 64;  // flip groups handled by the thread-per-row kernels

__device__ __forceinline__ double2 group_value(const CooGroup& g, const CooTerm* t, uint64_t col) {
    double re = 0.0, im = 0.0;
    for (int k = g.term_begin; k < g.term_end; ++k) {
        const bool neg = __popcll(col & t[k].z) & 1;
        re += neg ? -t[k].c_re : t[k].c_re;
        im += neg ? -t[k].c_im : t[k].c_im;
    }
    return make_double2(re, im);
}

__global__ void coo_count_kernel(const CooGroup* g, int n_groups, const CooTerm* t, uint64_t dim, int64_t* counts) {
    for (uint64_t row = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; row < dim;
         row += (uint64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        for (int q = 0; q < n_groups; ++q) {
            const double2 v = group_value(g[q], t, row ^ g[q].flip);
            c += (v.x != 0.0 || v.y != 0.0);
        }
        counts[row] = c;
    }
}

// thread per row: entries collected in local memory, insertion-sorted by column
__global__ void coo_write_kernel(const CooGroup* g, int n_groups, const CooTerm* t, uint64_t dim,
                                 const int64_t* offsets, int64_t* rows, int64_t* cols, double2* vals) {
    uint64_t kc[kThreadRowMax];
    double2 kv[kThreadRowMax];
    for (uint64_t row = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; row < dim;
         row += (uint64_t)gridDim.x * blockDim.x) {
        int m = 0;
        for (int q = 0; q < n_groups; ++q) {
            const uint64_t col = row ^ g[q].flip;
            const double2 v = group_value(g[q], t, col);
            if (v.x == 0.0 && v.y == 0.0) continue;
            int j = m++;
            while (j > 0 && kc[j - 1] > col) {
                kc[j] = kc[j - 1];
                kv[j] = kv[j - 1];
                --j;
            }
            kc[j] = col;
            kv[j] = v;
        }
        const int64_t o = offsets[row];
        for (int j = 0; j < m; ++j) {
            rows[o + j] = (int64_t)row;
            cols[o + j] = (int64_t)kc[j];
            vals[o + j] = kv[j];
        }
    }
}

// block per row for many flip groups: bitonic sort of (col, index) in shared memory
__global__ void coo_write_block_kernel(const CooGroup* g, int n_groups, const CooTerm* t, uint64_t dim,
                                       const int64_t* offsets, int64_t* rows, int64_t* cols, double2* vals) {
    extern __shared__ unsigned char smem[];
    const int P2 = 1 << (32 - __clz(n_groups - 1));  // next power of two
    uint64_t* key = reinterpret_cast<uint64_t*>(smem);
    int* idx = reinterpret_cast<int*>(key + P2);
    int* keep = idx + P2;
    for (uint64_t row = blockIdx.x; row < dim; row += gridDim.x) {
        for (int q = threadIdx.x; q < P2; q += blockDim.x) {
            key[q] = q < n_groups ? (row ^ g[q].flip) : ~0ull;
            idx[q] = q;
        }
        __syncthreads();
        for (int k = 2; k <= P2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < P2; i += blockDim.x) {
                    const int l = i ^ j;
                    if (l > i) {
                        const bool up = (i & k) == 0;
                        if ((key[i] > key[l]) == up) {
                            const uint64_t tk = key[i]; key[i] = key[l]; key[l] = tk;
                            const int ti = idx[i]; idx[i] = idx[l]; idx[l] = ti;
                        }
                    }
                }
                __syncthreads();
            }
        for (int q = threadIdx.x; q < n_groups; q += blockDim.x) {
            const double2 v = group_value(g[idx[q]], t, key[q]);
            keep[q] = (v.x != 0.0 || v.y != 0.0);
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // compaction in sorted order (n_groups entries)
            int64_t o = offsets[row];
            for (int q = 0; q < n_groups; ++q)
                if (keep[q]) {
                    rows[o] = (int64_t)row;
                    cols[o] = (int64_t)key[q];
                    vals[o] = group_value(g[idx[q]], t, key[q]);
                    ++o;
                }
        }
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_coo_count(const CooGroup* g, int n_groups, const CooTerm* t, int n, int64_t* counts,
                             cudaStream_t s) {
    const uint64_t dim = 1ull << n;
    const unsigned blocks = (unsigned)std::min<uint64_t>((dim + 255) / 256, 148 * 32);
    coo_count_kernel<<<blocks, 256, 0, s>>>(g, n_groups, t, dim, counts);
    return cudaGetLastError();
}

cudaError_t coo_scan(const int64_t* counts, int64_t* offsets, int64_t dim, void* scratch, size_t* scratch_bytes,
                     cudaStream_t s) {
    // offsets has dim + 1 entries: exclusive scan of counts followed by the total
    return cub::DeviceScan::ExclusiveSum(scratch, *scratch_bytes, counts, offsets, (int)(dim + 1), s);
}

cudaError_t launch_coo_write(const CooGroup* g, int n_groups, const CooTerm* t, int n, const int64_t* offsets,
                             int64_t* rows, int64_t* cols, double2* vals, cudaStream_t s) {
    const uint64_t dim = 1ull << n;
    if (n_groups <= kThreadRowMax) {
        const unsigned blocks = (unsigned)std::min<uint64_t>((dim + 127) / 128, 148 * 64);
        coo_write_kernel<<<blocks, 128, 0, s>>>(g, n_groups, t, dim, offsets, rows, cols, vals);
    } else {
        int p2 = 1;
        while (p2 < n_groups) p2 <<= 1;
        const size_t smem = (size_t)p2 * (8 + 4 + 4);
        const unsigned blocks = (unsigned)std::min<uint64_t>(dim, 148 * 16);
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(coo_write_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        coo_write_block_kernel<<<blocks, 256, smem, s>>>(g, n_groups, t, dim, offsets, rows, cols, vals);
    }
    return cudaGetLastError();
}

}  // namespace qfb
