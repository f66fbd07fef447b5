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

// Tiled kernels for <= 32 flip groups and n <= 31.  A thread owns one row: it
// evaluates the groups once (terms summed in input order, as the reference
// does), stages the non-zero values in group order, and ranks each entry's
// column without sorting: in flip order the rank is popc(m below q) plus the
// trie's difference-array events up to q (CooEvent; the list is uniform across
// the CTA, so this is straight-line integer work on the non-zero mask m).  The
// CTA's rows own one contiguous output range: a 16-bit (row in tile, group) key
// is staged at each entry's final position, and the range is stored coalesced
// with row, column and value rebuilt from the key.
constexpr int kTileRows = 128;
constexpr int kTileMaxTerms = 2048;

struct TileShared {
    int4 ev[96];            // (pos, d-bit, sign, mask)
    uint32_t flip[32];
    int2 range[32];         // term range per group
    uint32_t m[kTileRows];  // non-zero mask per row of the tile
    int base[kTileRows];    // first staged entry of the row
};

__device__ __forceinline__ void tile_setup(TileShared& sh, uint32_t* s_z, double2* s_c, const CooGroup* g,
                                           int n_groups, const CooTerm* t, int n_terms, const CooEvent* ev,
                                           int n_ev) {
    for (int i = threadIdx.x; i < n_ev; i += blockDim.x)
        sh.ev[i] = make_int4(ev[i].pos, (int)(1u << ev[i].d), ev[i].sign, (int)ev[i].mask);
    for (int i = threadIdx.x; i < n_groups; i += blockDim.x) {
        sh.flip[i] = (uint32_t)g[i].flip;
        sh.range[i] = make_int2(g[i].term_begin, g[i].term_end);
    }
    for (int i = threadIdx.x; i < n_terms; i += blockDim.x) {
        s_z[i] = (uint32_t)t[i].z;
        s_c[i] = make_double2(t[i].c_re, t[i].c_im);
    }
    __syncthreads();
}

__device__ __forceinline__ double2 tile_group_value(const TileShared& sh, const uint32_t* s_z, const double2* s_c,
                                                    int q, uint32_t col) {
    double re = 0.0, im = 0.0;
    const int2 r = sh.range[q];
    for (int k = r.x; k < r.y; ++k) {
        const double2 c = s_c[k];
        const bool neg = __popc(col & s_z[k]) & 1;
        re += neg ? -c.x : c.x;
        im += neg ? -c.y : c.y;
    }
    return make_double2(re, im);
}

__global__ void coo_count_tile_kernel(const CooGroup* g, int n_groups, const CooTerm* t, int n_terms, uint32_t dim,
                                      int64_t* counts) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ TileShared sh;
    double2* s_c = reinterpret_cast<double2*>(smem);
    uint32_t* s_z = reinterpret_cast<uint32_t*>(s_c + n_terms);
    tile_setup(sh, s_z, s_c, g, n_groups, t, n_terms, nullptr, 0);
    for (uint32_t row = blockIdx.x * blockDim.x + threadIdx.x; row < dim; row += gridDim.x * blockDim.x) {
        int c = 0;
        for (int q = 0; q < n_groups; ++q) {
            const double2 v = tile_group_value(sh, s_z, s_c, q, row ^ sh.flip[q]);
            c += (v.x != 0.0 || v.y != 0.0);
        }
        counts[row] = c;
    }
}

__global__ void __launch_bounds__(kTileRows) coo_write_tile_kernel(const CooGroup* g, int n_groups, const CooTerm* t,
                                                                   int n_terms, const CooEvent* ev, int n_ev,
                                                                   uint32_t dim, const int64_t* offsets,
                                                                   int64_t* rows, int64_t* cols, double2* vals) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ TileShared sh;
    double2* s_c = reinterpret_cast<double2*>(smem);
    double2* s_val = s_c + n_terms;
    uint32_t* s_z = reinterpret_cast<uint32_t*>(s_val + kTileRows * n_groups);
    uint16_t* s_key = reinterpret_cast<uint16_t*>(s_z + n_terms);
    tile_setup(sh, s_z, s_c, g, n_groups, t, n_terms, ev, n_ev);
    const uint32_t tiles = (dim + kTileRows - 1) / kTileRows;
    for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const uint32_t row0 = tile * kTileRows;
        const uint32_t row = row0 + threadIdx.x;
        const int64_t o0 = offsets[row0];
        const int64_t o1 = offsets[min(row0 + kTileRows, dim)];
        if (row < dim) {
            const int base = (int)(offsets[row] - o0);
            uint32_t m = 0;
            int c = 0;
            for (int q = 0; q < n_groups; ++q) {  // values in group order, compacted
                const double2 v = tile_group_value(sh, s_z, s_c, q, row ^ sh.flip[q]);
                if (v.x != 0.0 || v.y != 0.0) {
                    m |= 1u << q;
                    s_val[base + c++] = v;
                }
            }
            sh.m[threadIdx.x] = m;
            sh.base[threadIdx.x] = base;
            int acc = 0, e = 0;
            for (int q = 0; q < n_groups; ++q) {
                for (; e < n_ev; ++e) {
                    const int4 x = sh.ev[e];
                    if (x.x != q) break;
                    if (row & (uint32_t)x.y) acc += x.z * __popc(m & (uint32_t)x.w);
                }
                if ((m >> q) & 1) s_key[base + __popc(m & ((1u << q) - 1)) + acc] = (uint16_t)((threadIdx.x << 5) | q);
            }
        }
        __syncthreads();
        const int cnt = (int)(o1 - o0);
        for (int i = threadIdx.x; i < cnt; i += kTileRows) {
            const uint32_t key = s_key[i];
            const uint32_t rl = key >> 5, q = key & 31;
            const uint32_t r = row0 + rl;
            rows[o0 + i] = (int64_t)r;
            cols[o0 + i] = (int64_t)(r ^ sh.flip[q]);
            vals[o0 + i] = s_val[sh.base[rl] + __popc(sh.m[rl] & ((1u << q) - 1))];
        }
        __syncthreads();
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

template <typename V>
__global__ void __launch_bounds__(256) coo_energy_kernel(const int64_t* rows, const int64_t* cols, const double2* vals,
                                                         int64_t nnz, int64_t chunk, const V* psi, double* part) {
    __shared__ double red[8];
    const int64_t k0 = (int64_t)blockIdx.x * chunk;
    const int64_t k1 = min(k0 + chunk, nnz);
    double acc = 0.0;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const V a = psi[rows[k]], c = psi[cols[k]];
        const double2 v = vals[k];
        const double vr = v.x * (double)c.x - v.y * (double)c.y;  // v psi[c]
        const double vi = v.x * (double)c.y + v.y * (double)c.x;
        acc += (double)a.x * vr + (double)a.y * vi;              // Re(conj(psi[r]) v psi[c])
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

}  // namespace

int coo_energy_blocks(int64_t nnz) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((nnz + 8191) / 8192, 148 * 16));
}

cudaError_t launch_coo_energy(int prec, const int64_t* rows, const int64_t* cols, const double2* vals, int64_t nnz,
                              const void* psi, double* part, cudaStream_t s) {
    const int blocks = coo_energy_blocks(nnz);
    const int64_t chunk = (nnz + blocks - 1) / blocks;
    if (prec == 1)  // QF_C128
        coo_energy_kernel<double2><<<blocks, 256, 0, s>>>(rows, cols, vals, nnz, chunk, (const double2*)psi, part);
    else
        coo_energy_kernel<float2><<<blocks, 256, 0, s>>>(rows, cols, vals, nnz, chunk, (const float2*)psi, part);
    return cudaGetLastError();
}

bool coo_tile_ok(int n, int n_groups, int n_terms) { return n <= 31 && n_groups <= 32 && n_terms <= kTileMaxTerms; }

cudaError_t launch_coo_count(const CooGroup* g, int n_groups, const CooTerm* t, int n_terms, int n, int64_t* counts,
                             cudaStream_t s) {
    const uint64_t dim = 1ull << n;
    if (coo_tile_ok(n, n_groups, n_terms)) {
        const size_t smem = (size_t)n_terms * 20;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(coo_count_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
        }
        const unsigned blocks = (unsigned)std::min<uint64_t>((dim + 255) / 256, 148 * 8);
        coo_count_tile_kernel<<<blocks, 256, smem, s>>>(g, n_groups, t, n_terms, (uint32_t)dim, counts);
    } else {
        const unsigned blocks = (unsigned)std::min<uint64_t>((dim + 255) / 256, 148 * 32);
        coo_count_kernel<<<blocks, 256, 0, s>>>(g, n_groups, t, dim, counts);
    }
    return cudaGetLastError();
}

cudaError_t coo_scan(const int64_t* counts, int64_t* offsets, int64_t dim, void* scratch, size_t* scratch_bytes,
                     cudaStream_t s) {
    // offsets has dim + 1 entries: exclusive scan of counts followed by the total
    return cub::DeviceScan::ExclusiveSum(scratch, *scratch_bytes, counts, offsets, (int)(dim + 1), s);
}

cudaError_t launch_coo_write(const CooGroup* g, int n_groups, const CooTerm* t, int n_terms, const CooEvent* ev,
                             int n_ev, int n, const int64_t* offsets, int64_t* rows, int64_t* cols, double2* vals,
                             cudaStream_t s) {
    const uint64_t dim = 1ull << n;
    if (coo_tile_ok(n, n_groups, n_terms)) {
        const size_t smem = (size_t)kTileRows * n_groups * (16 + 2) + (size_t)n_terms * 20;
        cudaError_t e = cudaFuncSetAttribute(coo_write_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)std::max<size_t>(smem, 1));
        if (e != cudaSuccess) return e;
        const uint64_t tiles = (dim + kTileRows - 1) / kTileRows;
        const size_t per_cta = smem + sizeof(TileShared) + 1024;
        const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (227 * 1024) / per_cta));
        const unsigned blocks = (unsigned)std::min<uint64_t>(tiles, (uint64_t)148 * per_sm);
        coo_write_tile_kernel<<<blocks, kTileRows, smem, s>>>(g, n_groups, t, n_terms, ev, n_ev, (uint32_t)dim,
                                                              offsets, rows, cols, vals);
    } else if (n_groups <= kThreadRowMax) {
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
