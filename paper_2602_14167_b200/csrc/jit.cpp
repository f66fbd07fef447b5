// jit.cpp -- generator + NVRTC driver for the specialised sweep kernels.
// See jit.hpp.  The generated kernel does exactly what the AOT interpreter
// sweep_kernel<RT, R, BWD> (sweep_impl.cuh) does for one DevSweep, with every
// plan constant folded in.
#include "jit.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/file.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <set>
#include <mutex>
#include <sstream>
#include <thread>

#include "../../include/qforge_b200.h"

namespace qfb {

static const char* kPrelude =
#include "jit_prelude.inc"
    ;

namespace {

// ------------------------------------------------------------------ text
struct Out {
    std::string s;
    void operator()(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
        char buf[4096];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        s += buf;
        s += '\n';
    }
};


// Runtime or static value of memory bit `pos` for register index l in a phase.
struct BitSrc {
    int rb = -1;        // register bit (static)
    std::string expr;   // runtime expression (0/1), when rb < 0
};

// A per-thread condition: parity(tid & tm) ^ parity(tile_base & bm).  Used for
// deferred conditional relabelings: a cx whose control is a thread or tile bit
// (constant over the thread's registers) is not applied with selects per
// amplitude pair; the thread instead records "register label l holds amplitude
// l ^ (cond << t)" and conjugates the later gates on that bit by X (a few
// selects per gate), folding the relabeling into its store addresses.
struct Cond {
    uint32_t tm = 0, bm = 0;
    bool any() const { return tm || bm; }
    Cond& operator^=(const Cond& o) {
        tm ^= o.tm;
        bm ^= o.bm;
        return *this;
    }
};

std::string cond_expr(const Cond& c) {
    auto one = [](const char* v, uint32_t m) {
        if ((m & (m - 1)) == 0) {
            int j = __builtin_ctz(m);
            return std::string("((") + v + " >> " + std::to_string(j) + ") & 1u)";
        }
        return std::string("__popc(") + v + " & " + std::to_string(m) + "u)";
    };
    std::string e;
    if (c.tm) e = one("tid", c.tm);
    if (c.bm) e = e.empty() ? one("tile_base", c.bm) : "(" + e + " ^ " + one("tile_base", c.bm) + ")";
    if (e.empty()) return "0u";
    return "(" + e + " & 1u)";
}

// Per-sweep shared-memory swizzle: a linear map over GF(2) that fixes the low W
// bits of a tile index and adds to them, for each tile bit b >= W, a nonzero
// W-bit vector low[b] (the XOR-fold default is 1 << (b mod W)).  One wavefront
// serves the first W lane bits, so an exchange is bank-conflict free when those
// lanes' images are linearly independent in the low W bits; the default fails
// that for phases whose free tile bits miss a residue class mod W.  A
// hill-climb over low[] makes every phase of the sweep independent where it can
// (the default is kept when it already is, so such kernels are unchanged).
std::vector<uint32_t> sweep_swizzle(const PassPlan& pass, const DevSweep& sw, int W, bool search) {
    const int k = sw.k, R = sw.R, nl = std::min(W, k - R);
    std::vector<uint32_t> low(k, 0);
    for (int b = W; b < k; ++b) low[b] = 1u << (b % W);
    auto rank_ok = [&](const DevPhase& ph) {
        uint32_t rows[8];
        for (int j = 0; j < nl; ++j) {
            const int b = ph.thr_tl[j];
            rows[j] = b < W ? (1u << b) : low[b];
        }
        int rank = 0;
        for (int bit = 0; bit < W && rank < nl; ++bit) {
            int piv = -1;
            for (int j = rank; j < nl; ++j)
                if (rows[j] >> bit & 1) {
                    piv = j;
                    break;
                }
            if (piv < 0) continue;
            std::swap(rows[piv], rows[rank]);
            for (int j = 0; j < nl; ++j)
                if (j != rank && (rows[j] >> bit & 1)) rows[j] ^= rows[rank];
            ++rank;
        }
        return rank == nl;
    };
    auto bad = [&] {
        int c = 0;
        for (int f = 0; f < sw.n_phases; ++f) c += !rank_ok(pass.phases[sw.phase_begin + f]);
        return c;
    };
    int cur = bad();
    if (search && nl == W && cur > 0) {
        for (int round = 0; round < 8 && cur > 0; ++round) {
            bool improved = false;
            for (int b = W; b < k && cur > 0; ++b) {
                const uint32_t keep = low[b];
                uint32_t best_v = keep;
                for (uint32_t v = 1; v < (1u << W); ++v) {
                    low[b] = v;
                    const int c = bad();
                    if (c < cur) {
                        cur = c;
                        best_v = v;
                        improved = true;
                    }
                }
                low[b] = best_v;
            }
            if (!improved) break;
        }
    }
    std::vector<uint32_t> img(k);
    for (int b = 0; b < k; ++b) img[b] = (1u << b) | (b < W ? 0u : low[b]);
    return img;
}

// Development toggle (QF_CARVEOUT=1): all of L1 as shared memory.  Measured
// harmful (C2 light sweeps 7.0 -> 10.1 ms): the direct HBM loads need L1 for
// their in-flight lines, so the driver's default carveout is kept.
bool carveout_max() {
    const char* e = std::getenv("QF_CARVEOUT");
    return e && e[0] == '1';
}

bool env_flag(const char* name) {
    const char* e = std::getenv(name);
    return e && e[0] == '1';
}

}  // namespace

// Persistent cp.async double-buffered variant: QF_JIT_PIPE=1 for every sweep,
// QF_JIT_PIPE=light for sweeps of at most two phases (HBM-latency bound).
bool jit_pipe_mode(const PassPlan& pass, int si) {
    const char* e = std::getenv("QF_JIT_PIPE");
    if (!e) return false;
    if (e[0] == '1') return true;
    return std::strcmp(e, "light") == 0 && pass.sweeps[si].n_phases <= 2;
}

// QF_JIT_ILV=1: complex64 adjoint sweeps exchange psi and lambda as interleaved
// float4 pairs (one 128-bit STS/LDS per amplitude).  Measured slower on C2 (first
// adjoint sweep 64.4 -> 68.0 ms at batch 1024): the phases are FMA-pipe bound and
// the packing moves cost issue slots, so two float2 tiles stay the default.
bool jit_interleaved(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd) {
    return bwd && P.prec == QF_C64 && !jit_pipe_mode(pass, si) && env_flag("QF_JIT_ILV");
}

// Gradient taps are staged per thread in shared memory ([slots][T] reals) and
// reduced in batches at fixed points (no per-tap shuffle chains).
int jit_tap_stage(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd) {
    if (!bwd) return 0;
    int cap = P.prec == QF_C128 ? 16 : 32;
    if (const char* e = std::getenv("QF_JIT_TAPSTAGE")) cap = std::max(1, atoi(e));  // development (occupancy A/B)
    return std::min(pass.sweeps[si].n_taps, cap);
}

size_t jit_smem_bytes(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd) {
    const DevSweep& sw = pass.sweeps[si];
    const size_t vs = P.prec == QF_C128 ? 16 : 8;
    const int T = 1 << (sw.k - sw.R);
    const int nwarps = (T + 31) / 32;
    (void)nwarps;
    size_t b = ((size_t)1 << sw.k) * vs * (bwd ? 2 : 1) * (jit_pipe_mode(pass, si) ? 2 : 1);
    b += (size_t)((sw.n_mat + 1) & ~1) * vs;
    b += (size_t)jit_tap_stage(P, pass, si, bwd) * T * (vs / 2);
    return b;
}

std::string jit_source(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd) {
    const DevSweep& sw = pass.sweeps[si];
    const int k = sw.k, R = sw.R, NR = 1 << R, T = 1 << (k - R);
    const bool dbl = P.prec == QF_C128;
    // complex64 adjoint sweeps keep psi_p and lambda_p side by side in shared
    // memory (one 16-byte float4 per amplitude): every phase exchange is one
    // 128-bit STS + one 128-bit LDS per amplitude instead of two 64-bit each
    const bool ilv = jit_interleaved(P, pass, si, bwd);
    const int W = (dbl || ilv) ? 3 : 4;
    const char* Vt = dbl ? "double2" : "float2";
    const char* RTt = dbl ? "double" : "float";
    const int minb = [bwd] {
        const char* e = std::getenv(bwd ? "QF_JIT_MINB_BWD" : "QF_JIT_MINB_FWD");
        if (!e) e = std::getenv("QF_JIT_MINB");
        return e ? std::max(1, atoi(e)) : 2;
    }();
    const bool allow_direct = [] {
        const char* e = std::getenv("QF_JIT_DIRECT");
        return !(e && e[0] == '0');
    }();
    const bool allow_fuse = [] {
        const char* e = std::getenv("QF_JIT_FUSE");
        return !(e && e[0] == '0');
    }();
    const bool pipe = jit_pipe_mode(pass, si);
    // the sweep's shared-memory swizzle (the pipelined variant keeps the fold)
    const std::vector<uint32_t> img = sweep_swizzle(pass, sw, W, !pipe && !env_flag("QF_JIT_FOLDSWZ"));
    auto smap = [&](uint32_t p) {
        uint32_t r = 0;
        for (int b = 0; b < k; ++b)
            if (p >> b & 1) r ^= img[b];
        return r;
    };
    Out o;
    if (pipe) o.s += "// qf-option: pipelined\n";
    if (env_flag("QF_JIT_NOPACK")) o.s += "#define QF_NOPACK 1\n";
    o.s += kPrelude;
    o.s += "\n";
    o("namespace qfb {");
    const size_t decl_pos = o.s.size();  // namespace-scope tables are inserted here
    o("extern \"C\" __global__ void __launch_bounds__(%d, %d) qf_sweep(const SweepArgs a) {", T, minb);
    o("  typedef %s V; typedef %s RT;", Vt, RTt);
    const size_t sdecl_pos = o.s.size();  // function-scope static tables (diagonal-run products)
    o("  extern __shared__ __align__(16) unsigned char smem_raw[];");
    const unsigned TSZ = (1u << k) * (bwd ? 2u : 1u);  // one tile buffer (psi [+ lambda])
    const int S = jit_tap_stage(P, pass, si, bwd);
    const unsigned ntiles = 1u << (P.n - k);
    std::vector<uint32_t> joff(NR);
    for (int j = 0; j < NR; ++j) {
        uint32_t off = 0;
        for (int r = 0; r < R; ++r)
            if ((j >> r) & 1) off |= 1u << sw.tb[k - R + r];
        joff[j] = off;
    }
    if (!pipe) {
        o("  V* tile = reinterpret_cast<V*>(smem_raw);");
        o("  V* tile2 = tile + %u;", bwd ? (1u << k) : 0u);
        o("  V* smat = tile2 + %u;", 1u << k);
        if (ilv) o("  float4* tq = reinterpret_cast<float4*>(smem_raw); (void)tq;");
        o("  RT* stg = reinterpret_cast<RT*>(smat + %d);", (sw.n_mat + 1) & ~1);
        o("  (void)tile; (void)tile2; (void)stg;");
        o("  const uint32_t tid = threadIdx.x, tile_id = blockIdx.x; const int b = blockIdx.y;");
        o("  const uint32_t ntiles = gridDim.x;");
        o("  V* st = reinterpret_cast<V*>(a.psi) + (size_t)b * %zuull;", (size_t)1 << P.n);
        if (bwd) o("  V* lm = reinterpret_cast<V*>(a.lam) + (size_t)b * %zuull;", (size_t)1 << P.n);
        o("  const uint32_t tile_base = pdep_u32(tile_id, %uu);", sw.out_mask);
    } else {
        // Persistent CTA over a contiguous range of (state, tile) items; tile i+1 is
        // prefetched with cp.async into the second buffer while tile i is computed.
        o("  V* bufA = reinterpret_cast<V*>(smem_raw);");
        o("  V* bufB = bufA + %u;", TSZ);
        o("  V* smat = bufB + %u;", TSZ);
        o("  RT* stg = reinterpret_cast<RT*>(smat + %d);", (sw.n_mat + 1) & ~1);
        o("  (void)stg;");
        o("  const uint32_t tid = threadIdx.x;");
        o("  const uint32_t ntiles = %uu;", ntiles);
        o("  const long long items = (long long)%u * a.batch;", ntiles);
        o("  const long long per = (items + gridDim.x - 1) / gridDim.x;");
        o("  const long long it0 = (long long)blockIdx.x * per;");
        o("  const long long it1 = it0 + per < items ? it0 + per : items;");
        o("  if (it0 >= it1) return;");
        o("  uint32_t g_thr = 0;");
        for (int j = 0; j < k - R; ++j) o("  g_thr |= ((tid >> %d) & 1u) << %d;", j, sw.tb[j]);
        o("  auto prefetch = [&](V* buf, long long item) {");
        o("    const int pb = (int)(item >> %d);", P.n - k);
        o("    const uint32_t gb = pdep_u32((uint32_t)(item & %uu), %uu) | g_thr;", ntiles - 1, sw.out_mask);
        o("    const V* ps = reinterpret_cast<const V*>(a.psi) + (size_t)pb * %zuull;", (size_t)1 << P.n);
        if (bwd) o("    const V* pl = reinterpret_cast<const V*>(a.lam) + (size_t)pb * %zuull;", (size_t)1 << P.n);
        if (!bwd) {
            o("    if (a.from_zero) {");
            for (int j = 0; j < NR; ++j)
                o("      buf[swz<%d>(tid + %uu)] = mk_basis<V>((gb | %uu) == 0u);", W, (unsigned)(T * j), joff[j]);
            o("      return;");
            o("    }");
        }
        for (int j = 0; j < NR; ++j) {
            o("    cp_async_v(buf + swz<%d>(tid + %uu), ps + ((size_t)gb + %uull));", W, (unsigned)(T * j), joff[j]);
            if (bwd) o("    cp_async_v(buf + %u + swz<%d>(tid + %uu), pl + ((size_t)gb + %uull));", 1u << k, W, (unsigned)(T * j), joff[j]);
        }
        o("  };");
        o("  V* cur = bufA; V* nxt = bufB;");
        o("  prefetch(cur, it0);");
        o("  cp_async_commit();");
        o("  int cur_b = -1;");
        o("  for (long long it = it0; it < it1; ++it) {");
        o("  if (it + 1 < it1) prefetch(nxt, it + 1);");
        o("  cp_async_commit();");
        o("  cp_async_wait_1();");
        o("  __syncthreads();");
        o("  const int b = (int)(it >> %d); const uint32_t tile_id = (uint32_t)(it & %uu);", P.n - k, ntiles - 1);
        o("  V* tile = cur; V* tile2 = cur + %u; (void)tile2;", bwd ? (1u << k) : 0u);
        o("  V* st = reinterpret_cast<V*>(a.psi) + (size_t)b * %zuull;", (size_t)1 << P.n);
        if (bwd) o("  V* lm = reinterpret_cast<V*>(a.lam) + (size_t)b * %zuull;", (size_t)1 << P.n);
        o("  const uint32_t tile_base = pdep_u32(tile_id, %uu);", sw.out_mask);
        o("  if (b != cur_b) {");
        o("    const V* gm = reinterpret_cast<const V*>(a.gmat) + (size_t)b * a.gmat_stride + a.gmat_pass_base + %d;",
          sw.mbase);
        o("    for (int i = (int)tid; i < %d; i += %d) smat[i] = gm[i];", sw.n_mat, T);
        o("    cur_b = b;");
        o("    __syncthreads();");
        o("  }");
    }

    int tl_of_pos[64];
    for (int p = 0; p < 64; ++p) tl_of_pos[p] = -1;
    for (int t = 0; t < k; ++t) tl_of_pos[(int)sw.tb[t]] = t;
    const int nph = sw.n_phases;
    auto phase = [&](int f) -> const DevPhase& { return pass.phases[sw.phase_begin + f]; };
    // A phase can move its registers straight to/from HBM when its lanes cover the
    // lowest tile bits (>= 32-byte contiguous runs per lane group: full sectors).
    auto lanes_cover_low = [&](const DevPhase& ph) {
        if (T < 32) return true;
        const int need = dbl ? 1 : 2;
        int have = 0;
        for (int j = 0; j < 5 && j < k - R; ++j)
            if (ph.thr_tl[j] < need) ++have;
        return have == need;
    };
    // A phase change that keeps every warp-index thread bit (thread bits 5 and up)
    // on the same tile bit moves data only inside each warp's own region of the
    // tile: the region a warp stores before the change is exactly the one it loads
    // after it, so a __syncwarp orders it.  Warps may then run phases apart; two
    // warps in different phases of such a run still own disjoint regions (same
    // warp bits, different values), and every other change, the tap flushes and
    // the tile's final read-out stay CTA barriers.  (plan.cpp warp_bit_runs keeps
    // the warp bits fixed over runs of phases.)  QF_JIT_WARPSYNC=0: always barriers.
    static const bool warpsync_off = std::getenv("QF_JIT_WARPSYNC") && std::getenv("QF_JIT_WARPSYNC")[0] == '0';
    auto warp_local_exchange = [&](const DevPhase& a, const DevPhase* b) {
        if (warpsync_off || pipe || !b || T < 64) return false;
        for (int j = 5; j < k - R; ++j)
            if (a.thr_tl[j] != b->thr_tl[j]) return false;
        return true;
    };
    const bool direct_first = !pipe && allow_direct && nph > 0 && lanes_cover_low(phase(0));
    const bool direct_last = allow_direct && nph > 0 && lanes_cover_low(phase(nph - 1));
    // memory offset of register index l in phase f, and of the phase's thread base
    auto reg_goff = [&](const DevPhase& ph, int l) {
        uint32_t off = 0;
        for (int r = 0; r < R; ++r)
            if ((l >> r) & 1) off |= 1u << sw.tb[(int)ph.reg_tl[r]];
        return off;
    };
    auto emit_gbase = [&](const DevPhase& ph, const char* name) {
        o("  uint32_t %s = tile_base;", name);
        for (int j = 0; j < k - R; ++j) o("  %s |= ((tid >> %d) & 1u) << %d;", name, j, sw.tb[(int)ph.thr_tl[j]]);
    };

    if (!direct_first || !direct_last) {
        o("  uint32_t g_ld = tile_base;");
        for (int j = 0; j < k - R; ++j) o("  g_ld |= ((tid >> %d) & 1u) << %d;", j, sw.tb[j]);
    }
    if (pipe) {
        // loads / matrices handled in the loop header
    } else if (direct_first) {
        emit_gbase(phase(0), "g_p0");
        for (int l = 0; l < NR; ++l) {
            const uint32_t off = reg_goff(phase(0), l);
            if (!bwd)
                o("  V x%d = a.from_zero ? mk_basis<V>((g_p0 | %uu) == 0u) : st[(size_t)g_p0 + %uull];", l, off, off);
            else
                o("  V x%d = st[(size_t)g_p0 + %uull]; V y%d = lm[(size_t)g_p0 + %uull];", l, off, l, off);
        }
    } else {
        for (int j = 0; j < NR; ++j) {
            if (!bwd)
                o("  V v%d = a.from_zero ? mk_basis<V>((g_ld | %uu) == 0u) : st[(size_t)g_ld + %uull];", j, joff[j], joff[j]);
            else
                o("  V v%d = st[(size_t)g_ld + %uull]; V w%d = lm[(size_t)g_ld + %uull];", j, joff[j], j, joff[j]);
        }
    }
    if (!pipe) {
        o("  {  // this sweep's gate matrices (precomputed once per parameter set)");
        o("    const V* gm = reinterpret_cast<const V*>(a.gmat) + (size_t)b * a.gmat_stride + a.gmat_pass_base + %d;",
          sw.mbase);
        o("    for (int i = (int)tid; i < %d; i += %d) smat[i] = gm[i];", sw.n_mat, T);
    }
    // Uniform (per-state) products of a diagonal run's register-bit factors are
    // built once per CTA into shared memory, straight from the global matrix
    // table (the prologue is inserted here once every run is known; each entry
    // lists its factor indices), behind the same barrier as the matrices.
    const size_t stab_pos = o.s.size();
    if (!pipe) o("  }");
    // swizzled tile index of (tid, register j) in the load / read-out mapping
    auto emit_s_ld = [&] {
        o("  uint32_t s_ld = 0;");
        for (int j = 0; j < k - R; ++j) o("  s_ld ^= (0u - ((tid >> %d) & 1u)) & %uu;", j, smap(1u << j));
    };
    if (!direct_first && !pipe) {
        emit_s_ld();
        for (int j = 0; j < NR; ++j) {
            const unsigned c = smap((unsigned)(T * j));
            if (ilv)
                o("  tq[s_ld ^ %uu] = make_float4(v%d.x, v%d.y, w%d.x, w%d.y);", c, j, j, j, j);
            else if (bwd)
                o("  tile[s_ld ^ %uu] = v%d; tile2[s_ld ^ %uu] = w%d;", c, j, c, j);
            else
                o("  tile[s_ld ^ %uu] = v%d;", c, j);
        }
    }
    if (!pipe) o("  __syncthreads();");
    auto env_off = [](const char* name) {
        const char* e = std::getenv(name);
        return e && e[0] == '1';
    };
    const bool use_stab = !pipe && !env_off("QF_JIT_NOSTAB");  // development toggles (A/B, bisection)
    const bool use_ratio = bwd && !env_off("QF_JIT_NORATIO");
    const bool use_hoist = !env_off("QF_JIT_NOHOIST");
    const bool use_lazy = !env_off("QF_JIT_NOLAZY");
    const bool use_defer = !env_off("QF_JIT_NODEFER");
    std::vector<std::vector<int>> stab_entries;

    std::vector<const char*> arrs = {"x"};
    if (bwd) arrs.push_back("y");
    int uid = 0;  // unique names inside fused blocks
    auto emit_flush = [&](int first, int cnt, bool last = false) {
        o("    __syncthreads();");
        o("    tap_flush<RT>(stg, %d, %d, a.tap_part + ((size_t)b * a.n_taps_total + %d) * ntiles + tile_id, ntiles);",
          cnt, T, sw.tap_begin + first);
        if (!last) o("    __syncthreads();");  // the staging slots are reused
    };
    auto emit_flush_if_full = [&](int tap) {
        if (tap % S == S - 1) emit_flush(tap - (S - 1), S);
    };

    for (int f = 0; f < nph; ++f) {
        const DevPhase& ph = phase(f);
        int thr_of_tl[kMaxTileBits];
        for (int t = 0; t < kMaxTileBits; ++t) thr_of_tl[t] = -1;
        for (int j = 0; j < k - R; ++j) thr_of_tl[(int)ph.thr_tl[j]] = j;
        int rb_of_tl[kMaxTileBits];
        for (int t = 0; t < kMaxTileBits; ++t) rb_of_tl[t] = -1;
        for (int r = 0; r < R; ++r) rb_of_tl[(int)ph.reg_tl[r]] = r;
        auto src = [&](int pos) {
            BitSrc s;
            if (pos < 0) return s;
            int tl = pos < 64 ? tl_of_pos[pos] : -1;
            if (tl >= 0 && rb_of_tl[tl] >= 0) {
                s.rb = rb_of_tl[tl];
            } else if (tl >= 0) {
                s.expr = "((tid >> " + std::to_string(thr_of_tl[tl]) + ") & 1u)";
            } else {
                s.expr = "((tile_base >> " + std::to_string(pos) + ") & 1u)";
            }
            return s;
        };
        const bool dfirst = (f == 0 && direct_first);
        const bool dlast = (f == nph - 1 && direct_last);
        o("  { // phase %d%s%s", f, dfirst ? " (registers from HBM)" : "", dlast ? " (registers to HBM)" : "");
        std::vector<uint32_t> offs(NR);
        if (!dfirst || !dlast) {
            o("    uint32_t s_t = 0;");
            for (int j = 0; j < k - R; ++j)
                o("    s_t ^= (0u - ((tid >> %d) & 1u)) & %uu;", j, smap(1u << ph.thr_tl[j]));
            for (int l = 0; l < NR; ++l) {
                uint32_t off = 0;
                for (int r = 0; r < R; ++r)
                    if ((l >> r) & 1) off |= 1u << ph.reg_tl[r];
                offs[l] = smap(off);
            }
        }
        if (!dfirst) {
            for (int l = 0; l < NR; ++l) {
                if (ilv)
                    o("    V x%d, y%d; { const float4 q_ = tq[s_t ^ %uu]; x%d = make_float2(q_.x, q_.y); "
                      "y%d = make_float2(q_.z, q_.w); }", l, l, offs[l], l, l);
                else if (bwd)
                    o("    V x%d = tile[s_t ^ %uu]; V y%d = tile2[s_t ^ %uu];", l, offs[l], l, offs[l]);
                else
                    o("    V x%d = tile[s_t ^ %uu];", l, offs[l]);
            }
        }
        std::vector<int> phys(NR);
        for (int l = 0; l < NR; ++l) phys[l] = l;
        auto pairs = [&](int bit) {
            std::vector<std::pair<int, int>> v;
            for (int l = 0; l < NR; ++l)
                if (!((l >> bit) & 1)) v.push_back({phys[l], phys[l | (1 << bit)]});
            return v;
        };
        auto rename = [&](int tbit, int cbit) {  // cbit < 0: unconditional
            for (int l = 0; l < NR; ++l)
                if (!((l >> tbit) & 1) && (cbit < 0 || ((l >> cbit) & 1))) std::swap(phys[l], phys[l | (1 << tbit)]);
        };
        auto is_diagish = [&](uint8_t kd) { return kd == DK_D1 || kd == DK_D2 || kd == DK_TZ || kd == DK_TZZ; };
        // deferred conditional relabelings of the register bits (see Cond)
        std::vector<Cond> cond(R);
        auto ext_cond = [&](int pos) {  // condition "memory bit pos is 1" for a non-register bit
            Cond c;
            const int tl = pos < 64 ? tl_of_pos[pos] : -1;
            if (tl >= 0) c.tm = 1u << thr_of_tl[tl];
            else c.bm = 1u << pos;
            return c;
        };
        auto materialize = [&](int r) {  // apply a pending relabeling with selects
            if (r < 0 || !cond[r].any()) return;
            o("    { const bool c = %s != 0u;", cond_expr(cond[r]).c_str());
            for (const char* A : arrs)
                for (auto pr : pairs(r)) o("      jcswap(%s%d, %s%d, c);", A, pr.first, A, pr.second);
            o("    }");
            cond[r] = Cond{};
        };

        // ---- fused run of diagonal gates and Z-type taps (they all commute) ----
        auto flush_diag_run = [&](const std::vector<int>& run) {
            const int id = uid++;
            o("    { // fused diagonal run (%d ops)", (int)run.size());
            // taps first: v_l = Im(conj(lambda_l) psi_l) is invariant under diagonal
            // unitaries applied to both states, so every tap of the run shares it
            // Signed sums sum_l (-1)^{popc(l & mask)} v_l for every register-bit mask the
            // run's taps need come from one memoised Walsh tree (pair sums / differences
            // along register bit 0, then 1, ...); c64 keeps v_l as packed lane pairs
            // (FMUL2 / FADD2) and differences the lanes once per tap.
            std::map<int, std::string> wsum;
            {
                std::set<int> masks;
                for (int oi : run) {
                    const DevOp& op = pass.ops[oi];
                    if (op.kind != DK_TZ && op.kind != DK_TZZ) continue;
                    BitSrc s0 = src(op.pos0);
                    BitSrc s1 = op.kind == DK_TZZ ? src(op.pos1) : BitSrc{};
                    int m = 0;
                    if (s0.rb >= 0) m ^= 1 << s0.rb;
                    if (op.kind == DK_TZZ && s1.rb >= 0) m ^= 1 << s1.rb;
                    masks.insert(m);
                }
                if (!masks.empty()) {
                    const char* TT = dbl ? "RT" : "V";
                    std::vector<std::string> vec(NR);
                    for (int l = 0; l < NR; ++l) {
                        vec[l] = "v" + std::to_string(id) + "_" + std::to_string(l);
                        if (dbl)
                            o("      const RT %s = imcv(y%d, x%d);", vec[l].c_str(), phys[l], phys[l]);
                        else
                            o("      const V %s = jim2(y%d, x%d);", vec[l].c_str(), phys[l], phys[l]);
                    }
                    int wc = 0;
                    std::function<std::map<int, std::string>(const std::vector<std::string>&, const std::set<int>&)> walsh =
                        [&](const std::vector<std::string>& v, const std::set<int>& ms) {
                            std::map<int, std::string> res;
                            if (v.size() == 1) {
                                res[0] = v[0];
                                return res;
                            }
                            std::set<int> m0, m1;
                            for (int m : ms) ((m & 1) ? m1 : m0).insert(m >> 1);
                            for (int par = 0; par < 2; ++par) {
                                const std::set<int>& mm = par ? m1 : m0;
                                if (mm.empty()) continue;
                                std::vector<std::string> h(v.size() / 2);
                                for (size_t j = 0; j < h.size(); ++j) {
                                    h[j] = "w" + std::to_string(id) + "_" + std::to_string(wc++);
                                    if (dbl)
                                        o("      const RT %s = %s %c %s;", h[j].c_str(), v[2 * j].c_str(), par ? '-' : '+',
                                          v[2 * j + 1].c_str());
                                    else
                                        o("      const V %s = %s(%s, %s);", h[j].c_str(), par ? "jsub2" : "jadd2",
                                          v[2 * j].c_str(), v[2 * j + 1].c_str());
                                }
                                for (auto& kv : walsh(h, mm)) res[(kv.first << 1) | par] = kv.second;
                            }
                            return res;
                        };
                    for (auto& kv : walsh(vec, masks)) {
                        const std::string nm = "W" + std::to_string(id) + "_" + std::to_string(kv.first);
                        if (dbl)
                            o("      const RT %s = %s;", nm.c_str(), kv.second.c_str());
                        else
                            o("      const RT %s = %s.x - %s.y;", nm.c_str(), kv.second.c_str(), kv.second.c_str());
                        wsum[kv.first] = nm;
                    }
                    (void)TT;
                }
            }
            std::vector<std::string> rt_factors;                   // per-thread scalars
            std::vector<std::vector<std::pair<std::string, std::string>>> perbit(R);  // (f0, f1) per register bit
            std::vector<std::vector<std::pair<int, int>>> perbit_idx(R);  // their smat indices (-1: per-thread)
            struct D2s { int r0, r1; std::string d[4]; int moff = 0; };
            std::vector<D2s> d2s;
            for (size_t ri = 0; ri < run.size(); ++ri) {
                const int oi = run[ri];
                const DevOp& op = pass.ops[oi];
                const std::string nm = "f" + std::to_string(id) + "_" + std::to_string(ri);
                if (op.kind == DK_TZ || op.kind == DK_TZZ) {
                    BitSrc s0 = src(op.pos0);
                    BitSrc s1 = op.kind == DK_TZZ ? src(op.pos1) : BitSrc{};
                    int m = 0;
                    if (s0.rb >= 0) m ^= 1 << s0.rb;
                    if (op.kind == DK_TZZ && s1.rb >= 0) m ^= 1 << s1.rb;
                    o("      { RT s = %s;", wsum.at(m).c_str());
                    // sign: bits outside the registers, and relabeled register bits
                    Cond sc;
                    if (s0.rb < 0) sc ^= ext_cond(op.pos0);
                    else sc ^= cond[s0.rb];
                    if (op.kind == DK_TZZ) {
                        if (s1.rb < 0) sc ^= ext_cond(op.pos1);
                        else sc ^= cond[s1.rb];
                    }
                    if (sc.any()) o("        if (%s) s = -s;", cond_expr(sc).c_str());
                    o("        stg[%d * %d + tid] = s; }", op.tap % S, T);
                    emit_flush_if_full(op.tap);
                    continue;
                }
                if (op.kind == DK_D1) {
                    o("      const V %s_0 = smat[%d], %s_1 = smat[%d];", nm.c_str(), op.moff, nm.c_str(), op.moff + 1);
                    BitSrc s0 = src(op.pos0);
                    if (s0.rb >= 0) {
                        perbit[s0.rb].push_back({nm + "_0", nm + "_1"});
                        perbit_idx[s0.rb].push_back({op.moff, op.moff + 1});
                    } else
                        rt_factors.push_back("(" + s0.expr + " ? " + nm + "_1 : " + nm + "_0)");
                } else {  // DK_D2
                    o("      const V %s_0 = smat[%d], %s_1 = smat[%d], %s_2 = smat[%d], %s_3 = smat[%d];", nm.c_str(),
                      op.moff, nm.c_str(), op.moff + 1, nm.c_str(), op.moff + 2, nm.c_str(), op.moff + 3);
                    BitSrc s0 = src(op.pos0), s1 = src(op.pos1);
                    if (s0.rb < 0 && s1.rb < 0) {
                        rt_factors.push_back("(" + s0.expr + " ? (" + s1.expr + " ? " + nm + "_3 : " + nm + "_2) : (" +
                                             s1.expr + " ? " + nm + "_1 : " + nm + "_0))");
                    } else if (s0.rb >= 0 && s1.rb < 0) {
                        o("      const V %s_e0 = %s ? %s_1 : %s_0, %s_e1 = %s ? %s_3 : %s_2;", nm.c_str(), s1.expr.c_str(),
                          nm.c_str(), nm.c_str(), nm.c_str(), s1.expr.c_str(), nm.c_str(), nm.c_str());
                        perbit[s0.rb].push_back({nm + "_e0", nm + "_e1"});
                        perbit_idx[s0.rb].push_back({-1, -1});
                    } else if (s0.rb < 0 && s1.rb >= 0) {
                        o("      const V %s_e0 = %s ? %s_2 : %s_0, %s_e1 = %s ? %s_3 : %s_1;", nm.c_str(), s0.expr.c_str(),
                          nm.c_str(), nm.c_str(), nm.c_str(), s0.expr.c_str(), nm.c_str(), nm.c_str());
                        perbit[s1.rb].push_back({nm + "_e0", nm + "_e1"});
                        perbit_idx[s1.rb].push_back({-1, -1});
                    } else {
                        D2s d;
                        d.r0 = s0.rb;
                        d.r1 = s1.rb;
                        for (int q = 0; q < 4; ++q) d.d[q] = nm + "_" + std::to_string(q);
                        d.moff = op.moff;
                        d2s.push_back(d);
                    }
                }
            }
            // combine per-thread scalars
            const bool have_c = !rt_factors.empty();
            {
                std::vector<int> ubits;
                bool uniform = use_stab;
                for (int r = 0; r < R; ++r) {
                    bool used = !perbit[r].empty();
                    for (auto& d : d2s) used |= d.r0 == r || d.r1 == r;
                    if (used) ubits.push_back(r);
                    for (auto& pi : perbit_idx[r]) uniform &= pi.first >= 0;
                }
                uint32_t cbits = 0;  // ubits (by index) carrying a pending relabeling
                for (size_t bi = 0; bi < ubits.size(); ++bi)
                    if (cond[ubits[bi]].any()) cbits |= 1u << bi;
                if (!uniform || ubits.empty())
                    for (int r : ubits) materialize(r);  // per-thread tables index by label
                if (uniform && !ubits.empty()) {
                    // Adjoint pass: only conj(lambda) psi products are ever used, so each
                    // single-qubit diagonal may carry its own global phase: diag(d0, d1)
                    // is applied as diag(1, d1 conj(d0)) and amplitudes whose register
                    // bits are all 0 are left untouched (kRatio entries).
                    const int kRatio = 0x8000;
                    const int ne = 1 << ubits.size();
                    std::vector<int> slot(ne, -1);
                    if (cbits) {
                        // A relabeled bit either indexes the table at run time (dense: the
                        // identity entries are no longer skipped) or is materialised with
                        // selects first; pick the cheaper (FMA-pipe work weighs double).
                        int empties = 0;
                        if (use_ratio && !have_c && d2s.empty()) empties = 1;  // e = 0 only
                        const int extra = empties * (NR / ne) * (int)arrs.size();      // jcmul = 2 FMA-pipe instrs
                        const int fsel = __builtin_popcount(cbits) * 2 * NR * (int)arrs.size();
                        if (extra * 4 >= fsel) {
                            for (size_t bi = 0; bi < ubits.size(); ++bi)
                                if ((cbits >> bi) & 1u) materialize(ubits[bi]);
                            cbits = 0;
                        }
                    }
                    for (int e = 0; e < ne; ++e) {
                        std::vector<int> f;
                        for (size_t bi = 0; bi < ubits.size(); ++bi)
                            for (auto& pi : perbit_idx[ubits[bi]]) {
                                // Not combined with per-thread factors: at n = 30 (c64) that mix
                                // loses ~1e-4 on cancellation-dominated gradients (c128 exact).
                                if (use_ratio && !have_c) {
                                    if ((e >> bi) & 1) f.push_back(kRatio | pi.first);
                                } else {
                                    f.push_back(((e >> bi) & 1) ? pi.second : pi.first);
                                }
                            }
                        for (auto& d : d2s) {
                            const int i0 = (int)(std::find(ubits.begin(), ubits.end(), d.r0) - ubits.begin());
                            const int i1 = (int)(std::find(ubits.begin(), ubits.end(), d.r1) - ubits.begin());
                            f.push_back(d.moff + (((e >> i0) & 1) << 1 | ((e >> i1) & 1)));
                        }
                        if (f.empty() && !cbits) continue;  // identity (dense table when indexed at run time)
                        slot[e] = (int)stab_entries.size();
                        stab_entries.push_back(f);
                    }
                    if (cbits) {
                        std::string em;
                        for (size_t bi = 0; bi < ubits.size(); ++bi)
                            if ((cbits >> bi) & 1u)
                                em += (em.empty() ? "" : " | ") + std::string("(") + cond_expr(cond[ubits[bi]]) + " << " +
                                      std::to_string(bi) + ")";
                        o("      const uint32_t em%d = %s;", id, em.c_str());
                        for (int e = 0; e < ne; ++e) {
                            if (have_c) {
                                if (e == 0) {
                                    o("      V c%d = %s;", id, rt_factors[0].c_str());
                                    for (size_t q = 1; q < rt_factors.size(); ++q)
                                        o("      c%d = cmul(c%d, %s);", id, id, rt_factors[q].c_str());
                                }
                                o("      const V u%d_%d = jcmul(stab[%d + (%du ^ em%d)], c%d);", id, e, slot[0], e, id, id);
                            } else {
                                o("      const V u%d_%d = stab[%d + (%du ^ em%d)];", id, e, slot[0], e, id);
                            }
                        }
                        for (const char* A : arrs)
                            for (int l = 0; l < NR; ++l) {
                                int e = 0;
                                for (size_t bi = 0; bi < ubits.size(); ++bi)
                                    if ((l >> ubits[bi]) & 1) e |= 1 << bi;
                                o("      %s%d = jcmul(%s%d, u%d_%d);", A, phys[l], A, phys[l], id, e);
                            }
                        o("    }");
                        return;
                    }
                    if (have_c) {
                        o("      V c%d = %s;", id, rt_factors[0].c_str());
                        for (size_t q = 1; q < rt_factors.size(); ++q)
                            o("      c%d = cmul(c%d, %s);", id, id, rt_factors[q].c_str());
                    }
                    for (int e = 0; e < ne; ++e) {
                        if (slot[e] < 0) {
                            if (have_c) o("      const V u%d_%d = c%d;", id, e, id);
                        } else if (have_c) {
                            o("      const V u%d_%d = jcmul(stab[%d], c%d);", id, e, slot[e], id);
                        } else {
                            o("      const V u%d_%d = stab[%d];", id, e, slot[e]);
                        }
                    }
                    for (const char* A : arrs)
                        for (int l = 0; l < NR; ++l) {
                            int e = 0;
                            for (size_t bi = 0; bi < ubits.size(); ++bi)
                                if ((l >> ubits[bi]) & 1) e |= 1 << bi;
                            if (slot[e] < 0 && !have_c) continue;
                            o("      %s%d = jcmul(%s%d, u%d_%d);", A, phys[l], A, phys[l], id, e);
                        }
                    o("    }");
                    return;
                }
            }
            if (have_c) {
                o("      V c%d = %s;", id, rt_factors[0].c_str());
                for (size_t q = 1; q < rt_factors.size(); ++q) o("      c%d = cmul(c%d, %s);", id, id, rt_factors[q].c_str());
            }
            // combine factors per register bit
            std::vector<int> bits;
            std::vector<std::pair<std::string, std::string>> pb(R);
            std::vector<bool> ident(R, true);
            for (int r = 0; r < R; ++r) {
                bool used = !perbit[r].empty();
                for (auto& d : d2s) used |= d.r0 == r || d.r1 == r;
                if (!used) continue;
                bits.push_back(r);
                if (perbit[r].empty()) continue;
                ident[r] = false;
                std::string a0 = perbit[r][0].first, a1 = perbit[r][0].second;
                for (size_t q = 1; q < perbit[r].size(); ++q) {
                    const std::string n0 = "p" + std::to_string(id) + "_" + std::to_string(r) + "_" + std::to_string(q);
                    o("      const V %s_0 = cmul(%s, %s), %s_1 = cmul(%s, %s);", n0.c_str(), a0.c_str(),
                      perbit[r][q].first.c_str(), n0.c_str(), a1.c_str(), perbit[r][q].second.c_str());
                    a0 = n0 + "_0";
                    a1 = n0 + "_1";
                }
                pb[r] = {a0, a1};
            }
            if (!have_c && bits.empty()) {
                o("    }");
                return;
            }
            // table over the factor bits: entry index = bits of l restricted to `bits`
            std::vector<std::string> tab = {have_c ? ("c" + std::to_string(id)) : std::string()};
            int tcount = 0;
            for (size_t bi = 0; bi < bits.size(); ++bi) {
                const int r = bits[bi];
                std::vector<std::string> nt(tab.size() * 2);
                for (size_t e = 0; e < tab.size(); ++e) {
                    for (int v = 0; v < 2; ++v) {
                        const std::string fac = ident[r] ? std::string() : (v ? pb[r].second : pb[r].first);
                        std::string res;
                        if (tab[e].empty()) res = fac;
                        else if (fac.empty()) res = tab[e];
                        else {
                            res = "t" + std::to_string(id) + "_" + std::to_string(tcount++);
                            o("      const V %s = cmul(%s, %s);", res.c_str(), tab[e].c_str(), fac.c_str());
                        }
                        nt[e | (size_t(v) << bi)] = res;
                    }
                }
                tab.swap(nt);
            }
            auto tidx = [&](int l) {
                size_t e = 0;
                for (size_t bi = 0; bi < bits.size(); ++bi)
                    if ((l >> bits[bi]) & 1) e |= size_t(1) << bi;
                return e;
            };
            for (auto& d : d2s) {  // both bits in registers: multiply the table entries
                auto pos_in = [&](int r) { return (int)(std::find(bits.begin(), bits.end(), r) - bits.begin()); };
                const int i0 = pos_in(d.r0), i1 = pos_in(d.r1);
                for (size_t e = 0; e < tab.size(); ++e) {
                    const int q = (int)(((e >> i0) & 1) << 1 | ((e >> i1) & 1));
                    const std::string res = "t" + std::to_string(id) + "_" + std::to_string(tcount++);
                    if (tab[e].empty())
                        o("      const V %s = %s;", res.c_str(), d.d[q].c_str());
                    else
                        o("      const V %s = cmul(%s, %s);", res.c_str(), tab[e].c_str(), d.d[q].c_str());
                    tab[e] = res;
                }
            }
            for (const char* A : arrs)
                for (int l = 0; l < NR; ++l) {
                    const std::string& fac = tab[tidx(l)];
                    if (!fac.empty()) o("      %s%d = jcmul(%s%d, %s);", A, phys[l], A, phys[l], fac.c_str());
                }
            o("    }");
        };

        // Diagonal ops and Z-type taps are held back and fused into one run, which is
        // applied only when a later op acts non-diagonally on one of their qubits
        // (they commute with everything else, and a tap on qubit q is invariant
        // under gates on other qubits applied to both states) or at the phase end.
        // Tap ops flush pending taps first so the staging slots fill in order.
        std::vector<int> pend;
        uint64_t pend_pos = 0;
        bool pend_tap = false;
        auto reg_pos = [&](int rb) { return (uint64_t)1 << sw.tb[(int)ph.reg_tl[rb]]; };
        auto flush_pending = [&] {
            if (!pend.empty()) flush_diag_run(pend);
            pend.clear();
            pend_pos = 0;
            pend_tap = false;
        };
        // At a forced flush, later diagonal gates (not taps, whose staging order is
        // fixed) are hoisted into the run when nothing in between acts
        // non-diagonally on their qubits.
        std::vector<char> hoisted(ph.op_end - ph.op_begin, 0);
        auto op_touch = [&](const DevOp& x) {
            uint64_t t = 0;
            if (is_diagish(x.kind)) return t;
            if (x.rb0 >= 0) t |= reg_pos(x.rb0);
            if (x.kind == DK_G2 && x.rb1 >= 0) t |= reg_pos(x.rb1);
            return t;
        };
        auto diag_pos = [&](const DevOp& x) {
            uint64_t t = 0;
            if (x.pos0 >= 0) t |= (uint64_t)1 << x.pos0;
            if ((x.kind == DK_D2 || x.kind == DK_TZZ) && x.pos1 >= 0) t |= (uint64_t)1 << x.pos1;
            return t;
        };
        auto hoist_from = [&](int from) {
            uint64_t blocked = 0;
            for (int j = from; j < ph.op_end; ++j) {
                const DevOp& x = pass.ops[j];
                if ((x.kind == DK_D1 || x.kind == DK_D2) && !hoisted[j - ph.op_begin] && !(diag_pos(x) & blocked)) {
                    pend.push_back(j);
                    hoisted[j - ph.op_begin] = 1;
                }
                blocked |= op_touch(x);
            }
        };
        int oi = ph.op_begin;
        while (oi < ph.op_end) {
            const DevOp& op = pass.ops[oi];
            if (hoisted[oi - ph.op_begin]) {
                ++oi;
                continue;
            }
            if (allow_fuse && is_diagish(op.kind)) {
                pend.push_back(oi);
                if (op.pos0 >= 0) pend_pos |= (uint64_t)1 << op.pos0;
                if ((op.kind == DK_D2 || op.kind == DK_TZZ) && op.pos1 >= 0) pend_pos |= (uint64_t)1 << op.pos1;
                pend_tap |= op.kind == DK_TZ || op.kind == DK_TZZ;
                ++oi;
                continue;
            }
            if (!pend.empty()) {
                uint64_t touch = 0;
                if (op.rb0 >= 0) touch |= reg_pos(op.rb0);
                if (op.kind == DK_G2 && op.rb1 >= 0) touch |= reg_pos(op.rb1);
                const bool is_tap = op.kind == DK_TX || op.kind == DK_TY;
                if ((touch & pend_pos) || (is_tap && pend_tap) || !allow_fuse || !use_lazy) {
                    if (use_hoist) hoist_from(oi);
                    flush_pending();
                }
            }
            switch (op.kind) {
                case DK_G1: case DK_R1: case DK_RX: {
                    if (op.kind != DK_RX && cond[op.rb0].any()) {  // X G X = [[m3, m2], [m1, m0]]
                        o("    { const V a0 = smat[%d], a1 = smat[%d], a2 = smat[%d], a3 = smat[%d]; const bool cc = %s != 0u;",
                          op.moff, op.moff + 1, op.moff + 2, op.moff + 3, cond_expr(cond[op.rb0]).c_str());
                        o("      const V m0 = cc ? a3 : a0, m1 = cc ? a2 : a1, m2 = cc ? a1 : a2, m3 = cc ? a0 : a3;");
                    } else  // rx commutes with X
                    o("    { const V m0 = smat[%d], m1 = smat[%d], m2 = smat[%d], m3 = smat[%d]; (void)m1; (void)m2; (void)m3;",
                      op.moff, op.moff + 1, op.moff + 2, op.moff + 3);
                    for (const char* A : arrs)
                        for (auto pr : pairs(op.rb0)) {
                            if (op.kind == DK_RX)
                                o("      jrx(%s%d, %s%d, m0);", A, pr.first, A, pr.second);
                            else
                                o("      %s(%s%d, %s%d, m0, m1, m2, m3);", op.kind == DK_R1 ? "jr1" : "jg1", A,
                                  pr.first, A, pr.second);
                        }
                    o("    }");
                    break;
                }
                case DK_RS: {
                    if (cond[op.rb0].any())  // X R(theta) X = R(-theta): negate the shear parameters
                        o("    { V m0 = smat[%d]; if (%s) { m0.x = -m0.x; m0.y = -m0.y; }", op.moff,
                          cond_expr(cond[op.rb0]).c_str());
                    else
                    o("    { const V m0 = smat[%d];", op.moff);
                    for (const char* A : arrs)
                        for (auto pr : pairs(op.rb0)) o("      jrs(%s%d, %s%d, m0);", A, pr.first, A, pr.second);
                    o("    }");
                    break;
                }
                case DK_X1:
                    rename(op.rb0, -1);
                    break;
                case DK_CX:
                    if (op.rb1 >= 0) {
                        // X_c CX X_c = X_t CX: a relabeled control passes its condition to the target
                        cond[op.rb0] ^= cond[op.rb1];
                        rename(op.rb0, op.rb1);
                    } else if (use_defer) {
                        cond[op.rb0] ^= ext_cond(op.pos0);
                    } else {
                        BitSrc c = src(op.pos0);
                        o("    { const bool c = %s != 0u;", c.expr.c_str());
                        for (const char* A : arrs)
                            for (auto pr : pairs(op.rb0)) o("      jcswap(%s%d, %s%d, c);", A, pr.first, A, pr.second);
                        o("    }");
                    }
                    break;
                case DK_D1: case DK_D2: case DK_TZ: case DK_TZZ:
                    flush_diag_run(std::vector<int>{oi});
                    break;
                case DK_G2: {
                    materialize(op.rb0);
                    materialize(op.rb1);
                    o("    { const V* m = smat + %d;", op.moff);
                    const int e0 = 1 << op.rb0, e1 = 1 << op.rb1;
                    for (const char* A : arrs)
                        for (int l = 0; l < NR; ++l) {
                            if ((l & e0) || (l & e1)) continue;
                            o("      jg2(%s%d, %s%d, %s%d, %s%d, m);", A, phys[l], A, phys[l | e1], A, phys[l | e0], A,
                              phys[l | e0 | e1]);
                        }
                    o("    }");
                    break;
                }
                case DK_TX: case DK_TY: {
                    if (!dbl) {  // c64: packed lane-pair accumulators (2 FFMA2 per amplitude pair)
                        // two independent accumulator chains per sum (halves the FFMA2
                        // dependency depth), merged with one FADD2; the final lane
                        // combination is one FADD2 + one FADD
                        const auto prs = pairs(op.rb0);
                        const int na = (prs.size() >= 4 && !env_flag("QF_JIT_TAPACC1")) ? 2 : 1;
                        o("    { V P0, M0, P1, M1; (void)P1; (void)M1;");
                        for (size_t q = 0; q < prs.size(); ++q) {
                            const int f = prs[q].first, g = prs[q].second, ai = (int)(q % na);
                            const bool first = q < (size_t)na;
                            if (op.kind == DK_TX) {  // Im(conj(y_f) x_g) + Im(conj(y_g) x_f)
                                if (first) o("      P%d = jim2(y%d, x%d); M%d = jim2(y%d, x%d);", ai, f, g, ai, g, f);
                                else o("      P%d = jim2a(y%d, x%d, P%d); M%d = jim2a(y%d, x%d, M%d);", ai, f, g, ai, ai, g, f, ai);
                            } else {  // Re(conj(y_g) x_f) - Re(conj(y_f) x_g)
                                if (first) o("      P%d = jre2(y%d, x%d); M%d = jre2(y%d, x%d);", ai, g, f, ai, f, g);
                                else o("      P%d = jre2a(y%d, x%d, P%d); M%d = jre2a(y%d, x%d, M%d);", ai, g, f, ai, ai, f, g, ai);
                            }
                        }
                        if (na == 2) o("      P0 = jadd2(P0, P1); M0 = jadd2(M0, M1);");
                        if (op.kind == DK_TX) {
                            o("      const V S_ = jadd2(P0, M0);");
                            o("      stg[%d * %d + tid] = S_.x - S_.y; }", op.tap % S, T);
                        } else {
                            o("      const V D_ = jsub2(P0, M0); const RT t_ = D_.x + D_.y;");
                            if (cond[op.rb0].any())  // X Y X = -Y
                                o("      stg[%d * %d + tid] = %s ? -t_ : t_; }", op.tap % S, T, cond_expr(cond[op.rb0]).c_str());
                            else
                                o("      stg[%d * %d + tid] = t_; }", op.tap % S, T);
                        }
                        emit_flush_if_full(op.tap);
                        break;
                    }
                    o("    { RT s = 0;");
                    if (op.kind == DK_TX) {
                        for (auto pr : pairs(op.rb0))
                            o("      s += imcv(y%d, x%d) + imcv(y%d, x%d);", pr.first, pr.second, pr.second, pr.first);
                    } else {
                        for (auto pr : pairs(op.rb0))
                            o("      s += recv(y%d, x%d) - recv(y%d, x%d);", pr.second, pr.first, pr.first, pr.second);
                    }
                    if (op.kind == DK_TY && cond[op.rb0].any()) o("      if (%s) s = -s;", cond_expr(cond[op.rb0]).c_str());
                    o("      stg[%d * %d + tid] = s; }", op.tap % S, T);
                    emit_flush_if_full(op.tap);
                    break;
                }
                default:
                    break;
            }
            ++oi;
        }
        flush_pending();
        // pending relabelings become store-address XORs (register label l holds l ^ cond)
        std::string gx, sx;
        for (int r = 0; r < R; ++r) {
            if (!cond[r].any()) continue;
            const std::string c = cond_expr(cond[r]);
            gx += " ^ ((0u - " + c + ") & " + std::to_string(1u << sw.tb[(int)ph.reg_tl[r]]) + "u)";
            sx += " ^ ((0u - " + c + ") & " + std::to_string(smap(1u << ph.reg_tl[r])) + "u)";
        }
        if (dlast) {
            emit_gbase(ph, "g_pl");
            if (!gx.empty()) o("    const uint32_t g_x = 0u%s;", gx.c_str());
            for (int l = 0; l < NR; ++l) {
                const uint32_t off = reg_goff(ph, l);
                // 64-bit index arithmetic: a 32-bit `g | C` index with C * sizeof(V) >= 2^31
                // is miscompiled (the constant is split out of the address and wraps),
                // which corrupted n >= 29 states (tools/micro/sweep_harness.cu)
                const std::string a = gx.empty() ? "(size_t)g_pl + " + std::to_string(off) + "ull"
                                                 : "((size_t)g_pl + " + std::to_string(off) + "ull) ^ (size_t)g_x";
                if (bwd)
                    o("    st[%s] = x%d; lm[%s] = y%d;", a.c_str(), phys[l], a.c_str(), phys[l]);
                else
                    o("    st[%s] = x%d;", a.c_str(), phys[l]);
            }
            o("  }");
        } else {
            if (!sx.empty()) o("    const uint32_t s_w = s_t%s;", sx.c_str());
            const char* sb = sx.empty() ? "s_t" : "s_w";
            for (int l = 0; l < NR; ++l) {
                if (ilv)
                    o("    tq[%s ^ %uu] = make_float4(x%d.x, x%d.y, y%d.x, y%d.y);", sb, offs[l], phys[l], phys[l],
                      phys[l], phys[l]);
                else if (bwd)
                    o("    tile[%s ^ %uu] = x%d; tile2[%s ^ %uu] = y%d;", sb, offs[l], phys[l], sb, offs[l], phys[l]);
                else
                    o("    tile[%s ^ %uu] = x%d;", sb, offs[l], phys[l]);
            }
            o("    %s", warp_local_exchange(ph, f + 1 < nph ? &phase(f + 1) : nullptr) ? "__syncwarp();"
                                                                                     : "__syncthreads();");
            o("  }");
        }
    }
    if (!direct_last) {
        if (pipe) {
            for (int j = 0; j < NR; ++j) {
                if (bwd)
                    o("  const V v%d_o = tile[swz<%d>(tid + %uu)]; const V w%d_o = tile2[swz<%d>(tid + %uu)];", j, W,
                      (unsigned)(T * j), j, W, (unsigned)(T * j));
                else
                    o("  const V v%d_o = tile[swz<%d>(tid + %uu)];", j, W, (unsigned)(T * j));
            }
        } else {
            o("  {");
            emit_s_ld();
            for (int j = 0; j < NR; ++j) {
                const unsigned c = smap((unsigned)(T * j));
                if (ilv)
                    o("  V v%d_o, w%d_o; { const float4 q_ = tq[s_ld ^ %uu]; v%d_o = make_float2(q_.x, q_.y); "
                      "w%d_o = make_float2(q_.z, q_.w); }", j, j, c, j, j);
                else if (bwd)
                    o("  const V v%d_o = tile[s_ld ^ %uu]; const V w%d_o = tile2[s_ld ^ %uu];", j, c, j, c);
                else
                    o("  const V v%d_o = tile[s_ld ^ %uu];", j, c);
            }
        }
        for (int j = 0; j < NR; ++j) {
            if (bwd)
                o("  st[(size_t)g_ld + %uull] = v%d_o; lm[(size_t)g_ld + %uull] = w%d_o;", joff[j], j, joff[j], j);
            else
                o("  st[(size_t)g_ld + %uull] = v%d_o;", joff[j], j);
        }
        if (!pipe) o("  }");
    }
    if (bwd && sw.n_taps % std::max(S, 1) != 0) {
        const int rem = sw.n_taps % S;
        emit_flush(sw.n_taps - rem, rem, !pipe);
    }
    if (pipe) {
        o("  __syncthreads();");
        o("  { V* t_ = cur; cur = nxt; nxt = t_; }");
        o("  }");
    }
    o("}");
    o("}  // namespace qfb");
    if (!stab_entries.empty()) {
        size_t nf = 1;
        for (auto& f : stab_entries) nf = std::max(nf, f.size());
        const size_t ne = stab_entries.size();
        std::string decl = "__constant__ unsigned short qf_stab_f[" + std::to_string(ne) + "][" +
                           std::to_string(nf) + "] = {";
        for (size_t e = 0; e < ne; ++e) {
            decl += e ? ",{" : "{";
            for (size_t q = 0; q < nf; ++q) {
                if (q) decl += ",";
                decl += std::to_string(q < stab_entries[e].size() ? stab_entries[e][q] : 0xffff);
            }
            decl += "}";
        }
        decl += "};\n";
        char buf[1024];
        // The factors come from the sweep's matrix block once it sits in shared
        // memory (one barrier), not from global memory: a chain of dependent L2
        // loads per entry stalled every CTA's prologue for microseconds.
        snprintf(buf, sizeof buf,
                 "    __syncthreads();  // smat complete\n"
                 "    for (int e = (int)tid; e < %zu; e += %d) {  // diagonal-run tables (uniform per state)\n"
                 "      V acc; acc.x = 1; acc.y = 0;\n"
                 "#pragma unroll\n"
                 "      for (int q = 0; q < %zu; ++q) {\n"
                 "        const unsigned i = qf_stab_f[e][q];\n"
                 "        if (i == 0xffffu) break;\n"
                 "        if (i & 0x8000u) { V d0 = smat[i & 0x7fffu]; d0.y = -d0.y; acc = cmul(acc, cmul(smat[(i & 0x7fffu) + 1], d0)); }\n"
                 "        else acc = cmul(acc, smat[i]);\n"
                 "      }\n"
                 "      stab[e] = acc;\n"
                 "    }\n",
                 ne, T, nf);
        o.s.insert(stab_pos, buf);  // (stab_pos > sdecl_pos > decl_pos: insert back to front)
        o.s.insert(sdecl_pos, "  __shared__ __align__(16) V stab[" + std::to_string(ne) + "];\n");
        o.s.insert(decl_pos, decl);
    }
    return o.s;
}

// ------------------------------------------------------------------ H|psi>
// Specialised lambda = H psi + E = Re<psi|lambda> for one observable (same
// output-stationary tiling as hpsi_kernel in kernels.cu, whose AOT form stays the
// fallback).  Amplitude p = tid + T i of the tile: every term's sign splits into
// a per-thread part (thread bits, bits above the tile, parity(f & z)) and a
// compile-time part over the register index i.  Diagonal terms accumulate one
// per-thread coefficient per register-bit mask and are expanded once at the end;
// flips inside the registers read registers, flips of thread bits read the
// shared-memory copy of the (own or partner) tile, partner tiles above the tile
// are loaded into registers.
int jit_hpsi_threads(const ObservablePlan& O) {
    const int TS = 1 << O.kh;
    return TS < 256 ? TS : 256;
}

// QF_JIT_HPSI_TMA=1: partner tiles of the specialised H|psi> by TMA bulk copy,
// double-buffered on two mbarriers.  Measured slower than the default direct
// register loads (C2 H|psi> 6.83 vs 5.73 ms, C3 46.9 vs 43.6 ms: the per-group
// barrier costs more than the L2 latency it hides; tools/r2_t3.sh), so opt-in.
static bool jit_hpsi_tma(const ObservablePlan& O) {
    static const bool on = std::getenv("QF_JIT_HPSI_TMA") && std::getenv("QF_JIT_HPSI_TMA")[0] == '1';
    if (!on) return false;
    for (const DevGroup& g : O.groups)
        if (g.f_out) return true;
    return false;
}

size_t jit_hpsi_smem(const ObservablePlan& O, int prec) {
    const size_t vs = prec == QF_C128 ? 16 : 8;
    return (jit_hpsi_tma(O) ? ((size_t)3 << O.kh) * vs + 64 + 16 : ((size_t)2 << O.kh) * vs + 64);
}

std::string jit_hpsi_source(const ObservablePlan& O, int prec) {
    const bool dbl = prec == QF_C128;
    const int kh = O.kh, TS = 1 << kh, T = jit_hpsi_threads(O), NA = TS / T;
    int LT = 0;
    while ((1 << LT) < T) ++LT;
    const size_t N = (size_t)1 << O.n;
    Out o;
    if (env_flag("QF_JIT_NOPACK")) o.s += "#define QF_NOPACK 1\n";
    o.s += kPrelude;
    o.s += "\n";
    o("namespace qfb {");
    o("extern \"C\" __global__ void __launch_bounds__(%d, 2) qf_hpsi(const HArgs a) {", T);
    o("  typedef %s V; typedef %s RT;", dbl ? "double2" : "float2", dbl ? "double" : "float");
    o("  extern __shared__ __align__(16) unsigned char smem_raw[];");
    const bool tma = jit_hpsi_tma(O);
    o("  V* own = reinterpret_cast<V*>(smem_raw); V* part = own + %d; (void)own; (void)part;", TS);
    if (tma) {
        o("  V* part1 = part + %d;", TS);
        o("  double* red = reinterpret_cast<double*>(part1 + %d);", TS);
        o("  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 8);");
    } else {
        o("  double* red = reinterpret_cast<double*>(part + %d);", TS);
    }
    o("  const uint32_t tid = threadIdx.x, tile = blockIdx.x; const int b = blockIdx.y;");
    o("  const V* ps = reinterpret_cast<const V*>(a.psi) + (size_t)b * %zuull;", N);
    o("  const uint32_t base = tile << %d; (void)base;", kh);
    for (int i = 0; i < NA; ++i) o("  const V po%d = ps[(size_t)base + (tid + %uu)];", i, (unsigned)(T * i));
    std::vector<uint32_t> outer_f;  // outer groups in order (TMA prefetch chain)
    for (const DevGroup& g : O.groups)
        if (g.f_out) outer_f.push_back(g.f_out);
    const unsigned tile_bytes = (unsigned)TS * (dbl ? 16u : 8u);
    if (tma) {
        o("  if (tid == 0) { jit_mbar_init(&mbar[0]); jit_mbar_init(&mbar[1]); "
          "asm volatile(\"fence.mbarrier_init.release.cluster;\\n\" ::: \"memory\"); }");
        o("  __syncthreads();");
        o("  if (tid == 0) jit_bulk_load(part, ps + (size_t)(base ^ %uu), %uu, &mbar[0]);", outer_f[0], tile_bytes);
    }
    int outer_k = 0;
    bool own_smem = false;
    std::set<uint32_t> dmasks;
    for (const DevGroup& g : O.groups)
        for (int t = g.term_begin; t < g.term_end; ++t) {
            const DevTerm& d = O.terms[t];
            if (g.f_out == 0 && (d.f_in & (uint32_t)(T - 1))) own_smem = true;
            if (d.kind == TK_DIAG) dmasks.insert((d.z >> LT) & (uint32_t)(NA - 1));
        }
    if (own_smem) {
        for (int i = 0; i < NA; ++i) o("  own[tid + %uu] = po%d;", (unsigned)(T * i), i);
        o("  __syncthreads();");
    }
    for (int i = 0; i < NA; ++i) o("  V acc%d; acc%d.x = 0; acc%d.y = 0;", i, i, i);
    for (uint32_t m : dmasks) o("  RT dm%u = 0;", m);
    bool part_live = false;
    for (const DevGroup& g : O.groups) {
        const bool outer = g.f_out != 0;
        bool need_smem = false;
        for (int t = g.term_begin; t < g.term_end; ++t) need_smem |= (O.terms[t].f_in & (uint32_t)(T - 1)) != 0;
        o("  {  // flip group 0x%x", g.f_out);
        const char* pbuf = (outer_k & 1) ? "part1" : "part";
        if (outer && tma) {
            // this group's tile landed (buffer k & 1, phase k >> 1); every thread is done
            // with the other buffer (previous outer group), which takes the next tile
            o("    jit_mbar_wait(&mbar[%d], %uu);", outer_k & 1, (unsigned)((outer_k >> 1) & 1));
            o("    __syncthreads();");
            if (outer_k + 1 < (int)outer_f.size())
                o("    if (tid == 0) jit_bulk_load(%s, ps + (size_t)(base ^ %uu), %uu, &mbar[%d]);",
                  (outer_k & 1) ? "part" : "part1", outer_f[outer_k + 1], tile_bytes, (outer_k + 1) & 1);
            for (int i = 0; i < NA; ++i) o("    const V q%d = %s[tid + %uu];", i, pbuf, (unsigned)(T * i));
        } else if (outer) {
            for (int i = 0; i < NA; ++i)
                o("    const V q%d = ps[(size_t)(base ^ %uu) + (tid + %uu)];", i, g.f_out, (unsigned)(T * i));
            if (need_smem) {
                if (part_live) o("    __syncthreads();");
                for (int i = 0; i < NA; ++i) o("    part[tid + %uu] = q%d;", (unsigned)(T * i), i);
                o("    __syncthreads();");
                part_live = true;
            }
        }
        const char* R = outer ? "q" : "po";
        const char* S = outer ? (tma ? pbuf : "part") : "own";
        if (outer) ++outer_k;
        for (int t = g.term_begin; t < g.term_end; ++t) {
            const DevTerm& d = O.terms[t];
            const uint32_t zt = d.z & (uint32_t)(T - 1), zr = (d.z >> LT) & (uint32_t)(NA - 1);
            const uint32_t zh = d.z & ~(uint32_t)(TS - 1);
            const uint32_t ft = d.f_in & (uint32_t)(T - 1), fr = (d.f_in >> LT) & (uint32_t)(NA - 1);
            const double c = (d.kind != TK_DIAG && d.yodd) ? d.c_im : d.c_re;
            std::string sg;
            if (zt) sg += "__popc(tid & " + std::to_string(zt) + "u)";
            if (zh) sg += std::string(sg.empty() ? "" : " + ") + "__popc(base & " + std::to_string(zh) + "u)";
            if (d.fz_par & 1) sg += std::string(sg.empty() ? "" : " + ") + "1u";
            if (sg.empty())
                o("    { const RT k_ = (RT)(%.17g);", c);
            else
                o("    { const RT k_ = ((%s) & 1u) ? (RT)(%.17g) : (RT)(%.17g);", sg.c_str(), -c, c);
            if (d.kind == TK_DIAG) {
                o("      dm%u += k_; }", zr);
                continue;
            }
            if (zr) o("      const RT nk_ = -k_;");
            for (int i = 0; i < NA; ++i) {
                const bool neg = __builtin_popcount((unsigned)i & zr) & 1;
                char src[96];
                if (ft)
                    snprintf(src, sizeof src, "%s[(tid ^ %uu) + %uu]", S, ft, (unsigned)(T * ((unsigned)i ^ fr)));
                else
                    snprintf(src, sizeof src, "%s%u", R, (unsigned)i ^ fr);
                o("      acc%d = %s(%s, %s, acc%d);", i, d.yodd ? "jiaxpy" : "jaxpy", neg ? "nk_" : "k_", src, i);
            }
            o("    }");
        }
        o("  }");
    }
    if (!dmasks.empty())
        for (int i = 0; i < NA; ++i) {
            std::string e;
            for (uint32_t m : dmasks) {
                const bool neg = __builtin_popcount((unsigned)i & m) & 1;
                if (e.empty()) e = (neg ? "-dm" : "dm") + std::to_string(m);
                else e += (neg ? " - dm" : " + dm") + std::to_string(m);
            }
            o("  { const RT dg = %s; acc%d.x = fma(dg, po%d.x, acc%d.x); acc%d.y = fma(dg, po%d.y, acc%d.y); }",
              e.c_str(), i, i, i, i, i, i);
        }
    o("  double e = 0;");
    for (int i = 0; i < NA; ++i)
        o("  e += (double)po%d.x * (double)acc%d.x + (double)po%d.y * (double)acc%d.y;", i, i, i, i);
    o("  if (a.write_lam) {");
    o("    V* lm = reinterpret_cast<V*>(a.lam) + (size_t)b * %zuull;", N);
    for (int i = 0; i < NA; ++i) o("    lm[(size_t)base + (tid + %uu)] = acc%d;", (unsigned)(T * i), i);
    o("  }");
    o("  const unsigned m = lane_mask(%d);", T);
    o("  for (int off = %d; off > 0; off >>= 1) e += __shfl_xor_sync(m, e, off);", T >= 32 ? 16 : T / 2);
    o("  if ((tid & 31) == 0) red[tid >> 5] = e;");
    o("  __syncthreads();");
    o("  if (tid == 0) {");
    o("    double s = 0;");
    o("    for (int w = 0; w < %d; ++w) s += red[w];", (T + 31) / 32);
    o("    a.epart[(size_t)b * gridDim.x + tile] = s;");
    o("  }");
    o("}");
    o("}  // namespace qfb");
    return o.s;
}

// ------------------------------------------------------------------ NVRTC
namespace {

typedef int nvrtcResult;
typedef struct _nvrtcProgram* nvrtcProgram;
struct Nvrtc {
    void* h = nullptr;
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
    nvrtcResult (*logSize)(nvrtcProgram, size_t*);
    nvrtcResult (*log)(nvrtcProgram, char*);
    nvrtcResult (*cubinSize)(nvrtcProgram, size_t*);
    nvrtcResult (*cubin)(nvrtcProgram, char*);
    nvrtcResult (*destroy)(nvrtcProgram*);
    nvrtcResult (*version)(int*, int*);
    std::string err;
    bool load() {
        if (h) return true;
        const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                               "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_nvrtc/lib/libnvrtc.so.12"};
        for (const char* nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) {
            err = "NVRTC unavailable (libnvrtc.so.12 not found)";
            return false;
        }
        create = (decltype(create))dlsym(h, "nvrtcCreateProgram");
        compile = (decltype(compile))dlsym(h, "nvrtcCompileProgram");
        logSize = (decltype(logSize))dlsym(h, "nvrtcGetProgramLogSize");
        log = (decltype(log))dlsym(h, "nvrtcGetProgramLog");
        cubinSize = (decltype(cubinSize))dlsym(h, "nvrtcGetCUBINSize");
        cubin = (decltype(cubin))dlsym(h, "nvrtcGetCUBIN");
        destroy = (decltype(destroy))dlsym(h, "nvrtcDestroyProgram");
        version = (decltype(version))dlsym(h, "nvrtcVersion");
        if (!create || !compile || !logSize || !log || !cubinSize || !cubin || !destroy || !version) {
            err = "NVRTC library lacks required symbols";
            h = nullptr;
            return false;
        }
        return true;
    }
};
Nvrtc g_nvrtc;
std::mutex g_nvrtc_mu;

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

std::string cache_dir() {
    if (const char* e = std::getenv("QF_JIT_CACHE")) return e;
    const char* home = std::getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/qforge_b200";
}

void mkdirs(const std::string& d) {
    std::string cur;
    for (size_t i = 0; i < d.size(); ++i) {
        cur += d[i];
        if (d[i] == '/' && cur.size() > 1) mkdir(cur.c_str(), 0755);
    }
    mkdir(d.c_str(), 0755);
}

bool read_file(const std::string& p, std::string& out) {
    std::ifstream f(p, std::ios::binary);
    if (!f) return false;
    std::ostringstream ss;
    ss << f.rdbuf();
    out = ss.str();
    return !out.empty();
}

// Writes a cache entry atomically; a failed or short write is discarded.
void publish_cubin(const std::string& path, const std::string& cubin, const std::string& tag) {
    const std::string tmp = path + ".tmp" + std::to_string(getpid()) + tag;
    bool ok;
    {
        std::ofstream f(tmp, std::ios::binary);
        f.write(cubin.data(), (std::streamsize)cubin.size());
        f.flush();
        ok = f.good();
    }
    if (ok) ok = rename(tmp.c_str(), path.c_str()) == 0;
    if (!ok) unlink(tmp.c_str());
}

bool compile_one(const std::string& src, std::string& cubin, std::string& err) {
    if (const char* d = std::getenv("QF_JIT_DUMP")) {  // debugging: keep the generated source and cubin
        const std::string base = std::string(d) + "/qf_" + std::to_string(fnv1a(src));
        std::ofstream(base + ".cu") << src;
    }
    std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DQF_JIT=1"};
    // development: QF_JIT_OPTS = extra space-separated NVRTC options (A/B of compiler knobs)
    static const std::vector<std::string> extra = [] {
        std::vector<std::string> v;
        if (const char* e = std::getenv("QF_JIT_OPTS")) {
            std::istringstream is(e);
            std::string t;
            while (is >> t) v.push_back(t);
        }
        return v;
    }();
    for (const auto& x : extra) opts.push_back(x.c_str());
    nvrtcProgram prog = nullptr;
    if (g_nvrtc.create(&prog, src.c_str(), "qf_sweep.cu", 0, nullptr, nullptr) != 0) {
        err = "nvrtcCreateProgram failed";
        return false;
    }
    int rc = g_nvrtc.compile(prog, (int)opts.size(), opts.data());
    if (rc != 0) {
        size_t n = 0;
        g_nvrtc.logSize(prog, &n);
        std::string log(n, '\0');
        if (n) g_nvrtc.log(prog, &log[0]);
        err = "NVRTC compile failed: " + log.substr(0, 2000);
        g_nvrtc.destroy(&prog);
        return false;
    }
    size_t n = 0;
    g_nvrtc.cubinSize(prog, &n);
    cubin.assign(n, '\0');
    g_nvrtc.cubin(prog, &cubin[0]);
    g_nvrtc.destroy(&prog);
    return true;
}

// ---- process-wide module table (see jit.hpp) ----
struct Module {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    int refs = 0;
};
std::map<std::string, Module> g_modules;
std::mutex g_modules_mu;

// Loads (or shares) the module of `key`; false + err on failure (the caller
// treats a cached cubin that fails to load as corrupt).
bool module_acquire(const std::string& key, const std::string& cubin, const char* name, cudaKernel_t& kern,
                    std::string& err) {
    std::lock_guard<std::mutex> lk(g_modules_mu);
    auto it = g_modules.find(key);
    if (it != g_modules.end()) {
        it->second.refs++;
        kern = it->second.kern;
        return true;
    }
    Module m;
    cudaError_t e = cudaLibraryLoadData(&m.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
        return false;
    }
    e = cudaLibraryGetKernel(&m.kern, m.lib, name);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaLibraryUnload(m.lib);
        err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
        return false;
    }
    m.refs = 1;
    kern = m.kern;
    g_modules[key] = m;
    return true;
}

struct Job {
    const ProgramPlan* P;
    const PassPlan* pass;
    int si;
    bool bwd;
    std::string cubin, err;
    bool from_cache = false;
};

}  // namespace

void jit_release(JitKernel& k) {
    if (k.module.empty()) return;
    std::lock_guard<std::mutex> lk(g_modules_mu);
    auto it = g_modules.find(k.module);
    if (it != g_modules.end() && --it->second.refs == 0) {
        cudaLibraryUnload(it->second.lib);
        g_modules.erase(it);
    }
    k.module.clear();
    k.kernel = nullptr;
}

void jit_release(std::vector<JitKernel>& ks) {
    for (auto& k : ks) jit_release(k);
}

bool jit_compile_source(const std::string& src, std::string& cubin, std::string& err) {
    {
        std::lock_guard<std::mutex> lk(g_nvrtc_mu);
        if (!g_nvrtc.load()) {
            err = g_nvrtc.err;
            return false;
        }
    }
    return compile_one(src, cubin, err);
}

bool jit_build(const ProgramPlan& P, JitPass& fwd, JitPass& bwd, JitStats& st, bool load_modules) {
    auto t0 = std::chrono::steady_clock::now();
    {
        std::lock_guard<std::mutex> lk(g_nvrtc_mu);
        if (!g_nvrtc.load()) {
            st.error = g_nvrtc.err;
            return false;
        }
    }
    int maj = 0, min = 0;
    g_nvrtc.version(&maj, &min);
    std::vector<Job> jobs;
    for (size_t i = 0; i < P.fwd.sweeps.size(); ++i) jobs.push_back({&P, &P.fwd, (int)i, false, {}, {}, false});
    for (size_t i = 0; i < P.bwd.sweeps.size(); ++i) jobs.push_back({&P, &P.bwd, (int)i, true, {}, {}, false});
    const std::string dir = cache_dir();
    mkdirs(dir);
    // Several processes (one per GPU under torchrun) build the same program at
    // once: each source is claimed across processes with an O_EXCL lock file
    // next to its cache entry, so every kernel is compiled once per host and
    // the other processes pick up the cubin.  Pass 1 compiles what this
    // process claims and defers what another holds; pass 2 waits for those
    // (bounded; a stale or abandoned claim is compiled here instead).
    std::vector<std::string> srcs(jobs.size()), paths(jobs.size());
    std::vector<size_t> deferred;
    std::mutex def_mu;
    auto publish = [&](size_t j) { publish_cubin(paths[j], jobs[j].cubin, "_" + std::to_string(j)); };
    std::atomic<size_t> next{0};
    auto worker = [&] {
        for (;;) {
            size_t j = next.fetch_add(1);
            if (j >= jobs.size()) return;
            Job& jb = jobs[j];
            srcs[j] = jit_source(*jb.P, *jb.pass, jb.si, jb.bwd);
            char key[64];
            snprintf(key, sizeof key, "%016llx_%d_%d", (unsigned long long)fnv1a(srcs[j]), maj, min);
            paths[j] = dir + "/" + key + ".cubin";
            if (read_file(paths[j], jb.cubin)) {
                jb.from_cache = true;
                continue;
            }
            // claim: an advisory flock on the lock file (released by the kernel if
            // the holder dies, so an abandoned claim never stalls later builds)
            const std::string lock = paths[j] + ".lock";
            const int fd = open(lock.c_str(), O_CREAT | O_RDWR, 0644);
            if (fd >= 0 && flock(fd, LOCK_EX | LOCK_NB) != 0) {
                close(fd);
                std::lock_guard<std::mutex> lk(def_mu);
                deferred.push_back(j);
                continue;
            }
            if (!read_file(paths[j], jb.cubin)) {  // re-check under the claim
                if (compile_one(srcs[j], jb.cubin, jb.err)) publish(j);
            } else {
                jb.from_cache = true;
            }
            if (fd >= 0) {
                flock(fd, LOCK_UN);
                close(fd);
            }
        }
    };
    unsigned nthr = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("QF_JIT_THREADS")) nthr = (unsigned)std::max(1, atoi(e));
    nthr = std::max(1u, std::min<unsigned>(nthr, (unsigned)jobs.size()));
    std::vector<std::thread> pool;
    for (unsigned i = 0; i < nthr; ++i) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    pool.clear();
    next = 0;
    auto waiter = [&] {
        for (;;) {
            size_t d = next.fetch_add(1);
            if (d >= deferred.size()) return;
            const size_t j = deferred[d];
            Job& jb = jobs[j];
            // wait for the holder's claim (blocking flock: returns when it finishes or dies)
            const std::string lock = paths[j] + ".lock";
            const int fd = open(lock.c_str(), O_CREAT | O_RDWR, 0644);
            if (fd >= 0) flock(fd, LOCK_EX);
            if (read_file(paths[j], jb.cubin)) {
                jb.from_cache = true;
            } else if (compile_one(srcs[j], jb.cubin, jb.err)) {  // holder failed: reproduce the error here
                publish(j);
            }
            if (fd >= 0) {
                flock(fd, LOCK_UN);
                close(fd);
            }
        }
    };
    nthr = std::max(1u, std::min<unsigned>(nthr, (unsigned)std::max<size_t>(1, deferred.size())));
    for (unsigned i = 0; i < nthr && !deferred.empty(); ++i) pool.emplace_back(waiter);
    for (auto& t : pool) t.join();
    if (!load_modules) {  // compile / cache stage only (host-side check, no device needed)
        for (auto& jb : jobs) {
            if (!jb.err.empty()) {
                st.error = jb.err;
                return false;
            }
            if (jb.from_cache) st.cached++;
            else st.compiled++;
        }
        st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return true;
    }
    fwd.sweeps.assign(P.fwd.sweeps.size(), {});
    bwd.sweeps.assign(P.bwd.sweeps.size(), {});
    auto fail = [&](const std::string& e) {  // releases every module acquired so far
        st.error = e;
        jit_release(fwd.sweeps);
        jit_release(bwd.sweeps);
        return false;
    };
    for (auto& jb : jobs) {
        if (!jb.err.empty()) return fail(jb.err);
        cudaKernel_t kern;
        std::string lerr;
        const size_t jidx = (size_t)(&jb - jobs.data());
        if (!module_acquire(paths[jidx], jb.cubin, "qf_sweep", kern, lerr)) {
            // a truncated / corrupt cache entry: drop it and compile afresh
            unlink(paths[jidx].c_str());
            if (!jb.from_cache || !compile_one(srcs[jidx], jb.cubin, jb.err)) return fail(jb.err.empty() ? lerr : jb.err);
            publish(jidx);
            jb.from_cache = false;
            if (!module_acquire(paths[jidx], jb.cubin, "qf_sweep", kern, lerr)) return fail(lerr);
        }
        JitKernel& jk = (jb.bwd ? bwd : fwd).sweeps[jb.si];
        jk.kernel = (void*)kern;
        jk.module = paths[jidx];
        const DevSweep& sw = jb.pass->sweeps[jb.si];
        jk.threads = 1 << (sw.k - sw.R);
        jk.smem = jit_smem_bytes(P, *jb.pass, jb.si, jb.bwd);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, (const void*)kern);
        if (carveout_max())
            cudaFuncSetAttribute((const void*)kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (jk.smem + fa.sharedSizeBytes > 48 * 1024) {  // static tables count against the 48 KB default
            const cudaError_t e =
                cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jk.smem);
            if (e != cudaSuccess) return fail(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        }
        jk.pipe = jit_pipe_mode(*jb.pass, jb.si);
        if (jk.pipe) {
            int dev = 0, sms = 148, per = 1;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)kern, jk.threads, jk.smem) != cudaSuccess ||
                per < 1)
                per = 1;
            jk.ctas = sms * per;
        }
        if (jb.from_cache) st.cached++;
        else st.compiled++;
    }
    fwd.ok = bwd.ok = true;
    st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return true;
}

bool jit_build_hpsi(const ObservablePlan& O, int prec, JitKernel& out, std::string& err) {
    {
        std::lock_guard<std::mutex> lk(g_nvrtc_mu);
        if (!g_nvrtc.load()) {
            err = g_nvrtc.err;
            return false;
        }
    }
    int maj = 0, min = 0;
    g_nvrtc.version(&maj, &min);
    const std::string src = jit_hpsi_source(O, prec);
    const std::string dir = cache_dir();
    mkdirs(dir);
    char key[64];
    snprintf(key, sizeof key, "%016llx_%d_%d", (unsigned long long)fnv1a(src), maj, min);
    const std::string path = dir + "/" + key + ".cubin";
    std::string cubin;
    bool cached = read_file(path, cubin);
    if (!cached) {
        if (!compile_one(src, cubin, err)) return false;
        publish_cubin(path, cubin, "");
    }
    cudaKernel_t kern;
    if (!module_acquire(path, cubin, "qf_hpsi", kern, err)) {
        unlink(path.c_str());  // corrupt cache entry: recompile once
        if (!cached || !compile_one(src, cubin, err)) return false;
        publish_cubin(path, cubin, "");
        if (!module_acquire(path, cubin, "qf_hpsi", kern, err)) return false;
    }
    cudaError_t e;
    jit_release(out);
    out.kernel = (void*)kern;
    out.module = path;
    out.threads = jit_hpsi_threads(O);
    out.smem = jit_hpsi_smem(O, prec);
    if (carveout_max())
        cudaFuncSetAttribute((const void*)kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (out.smem > 48 * 1024) {
        e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out.smem);
        if (e != cudaSuccess) {
            err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
            return false;
        }
    }
    return true;
}

int jit_launch_hpsi(const JitKernel& k, const HArgs& a, int tiles, int batch, void* stream) {
    HArgs aa = a;
    void* args[] = {&aa};
    return (int)cudaLaunchKernel((const void*)k.kernel, dim3(tiles, batch), dim3(k.threads), args, k.smem,
                                 (cudaStream_t)stream);
}

thread_local std::string g_launch_detail;
const std::string& jit_last_launch_detail() { return g_launch_detail; }

int jit_launch(const JitKernel& k, const SweepArgs& a, int tiles, int batch, void* stream) {
    SweepArgs aa = a;
    aa.batch = batch;
    void* args[] = {&aa};
    dim3 grid(tiles, batch);
    if (k.pipe) {
        const long long items = (long long)tiles * batch;
        grid = dim3((unsigned)std::min<long long>(items, (long long)k.ctas));
    }
    cudaError_t e = cudaLaunchKernel((const void*)k.kernel, grid, dim3(k.threads), args, k.smem, (cudaStream_t)stream);
    if (e != cudaSuccess) {  // keep the launch configuration next to the error for diagnosis
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, (const void*)k.kernel);
        char buf[320];
        snprintf(buf, sizeof buf,
                 "sweep launch grid (%u, %u) x %d threads, dynamic smem %zu B; kernel: %d regs, static smem %zu B, "
                 "local %zu B, max threads %d, max dynamic smem %d B",
                 grid.x, grid.y, k.threads, k.smem, fa.numRegs, fa.sharedSizeBytes, fa.localSizeBytes,
                 fa.maxThreadsPerBlock, fa.maxDynamicSharedSizeBytes);
        g_launch_detail = buf;
    }
    return (int)e;
}

}  // namespace qfb
