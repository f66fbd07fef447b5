// jit.cpp -- generator + NVRTC driver for the specialised sweep kernels.
// See jit.hpp.  The generated kernel does exactly what the AOT interpreter
// sweep_kernel<RT, R, BWD> (sweep_impl.cuh) does for one DevSweep, with every
// plan constant folded in.
#include "jit.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
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

uint32_t swz_host(uint32_t p, int W) {
    uint32_t x = p >> W, f = 0;
    for (int i = 0; i < 4; ++i) {
        f ^= x;
        x >>= W;
    }
    return p ^ (f & ((1u << W) - 1));
}

// Runtime or static value of memory bit `pos` for register index l in a phase.
struct BitSrc {
    int rb = -1;        // register bit (static)
    std::string expr;   // runtime expression (0/1), when rb < 0
};

}  // namespace

size_t jit_smem_bytes(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd) {
    const DevSweep& sw = pass.sweeps[si];
    const size_t vs = P.prec == QF_C128 ? 16 : 8;
    const int T = 1 << (sw.k - sw.R);
    const int nwarps = (T + 31) / 32;
    size_t b = ((size_t)1 << sw.k) * vs * (bwd ? 2 : 1);
    b += (size_t)((sw.n_mat + 1) & ~1) * vs;
    b += (size_t)sw.n_taps * nwarps * 8;
    return b;
}

std::string jit_source(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd) {
    const DevSweep& sw = pass.sweeps[si];
    const int k = sw.k, R = sw.R, NR = 1 << R, T = 1 << (k - R);
    const int nwarps = (T + 31) / 32;
    const bool dbl = P.prec == QF_C128;
    const int W = dbl ? 3 : 4;
    const char* Vt = dbl ? "double2" : "float2";
    const char* RTt = dbl ? "double" : "float";
    const int minb = [] {
        const char* e = std::getenv("QF_JIT_MINB");
        return e ? std::max(1, atoi(e)) : 1;
    }();
    Out o;
    o.s += kPrelude;
    o.s += "\n";
    o("namespace qfb {");
    o("extern \"C\" __global__ void __launch_bounds__(%d, %d) qf_sweep(const SweepArgs a) {", T, minb);
    o("  typedef %s V; typedef %s RT;", Vt, RTt);
    o("  extern __shared__ __align__(16) unsigned char smem_raw[];");
    o("  V* tile = reinterpret_cast<V*>(smem_raw);");
    o("  V* tile2 = tile + %u;", bwd ? (1u << k) : 0u);
    o("  V* smat = tile2 + %u;", 1u << k);
    o("  double* stap = reinterpret_cast<double*>(smat + %d);", (sw.n_mat + 1) & ~1);
    o("  (void)tile2; (void)stap;");
    o("  const uint32_t tid = threadIdx.x, tile_id = blockIdx.x; const int b = blockIdx.y;");
    o("  V* st = reinterpret_cast<V*>(a.psi) + (size_t)b * %zuull;", (size_t)1 << P.n);
    if (bwd) o("  V* lm = reinterpret_cast<V*>(a.lam) + (size_t)b * %zuull;", (size_t)1 << P.n);
    o("  const uint32_t tile_base = pdep_u32(tile_id, %uu);", sw.out_mask);
    o("  uint32_t g_ld = tile_base;");
    for (int j = 0; j < k - R; ++j) o("  g_ld |= ((tid >> %d) & 1u) << %d;", j, sw.tb[j]);
    std::vector<uint32_t> joff(NR);
    for (int j = 0; j < NR; ++j) {
        uint32_t off = 0;
        for (int r = 0; r < R; ++r)
            if ((j >> r) & 1) off |= 1u << sw.tb[k - R + r];
        joff[j] = off;
    }
    // HBM -> registers (all loads in flight), then prologue, then registers -> shared
    for (int j = 0; j < NR; ++j) {
        if (!bwd)
            o("  V v%d = a.from_zero ? mk_basis<V>((g_ld | %uu) == 0u) : st[g_ld | %uu];", j, joff[j], joff[j]);
        else
            o("  V v%d = st[g_ld | %uu]; V w%d = lm[g_ld | %uu];", j, joff[j], j, joff[j]);
    }
    o("  {");
    o("    const double* th = a.theta + (size_t)(b + a.batch_offset) * a.P;");
    o("    for (int op_i = %d + (int)tid; op_i < %d; op_i += %d) {", sw.op_begin, sw.op_end, T);
    o("      const DevOp op = a.ops[op_i];");
    o("      if (op.moff >= 0) build_matrix<V, %s>(op, a.gates[op.gate], th, a.cmats, smat + op.moff);",
      bwd ? "true" : "false");
    o("    }");
    o("  }");
    for (int j = 0; j < NR; ++j) {
        o("  tile[swz<%d>(tid + %uu)] = v%d;%s", W, (unsigned)(T * j), j,
          bwd ? (" tile2[swz<" + std::to_string(W) + ">(tid + " + std::to_string(T * j) + "u)] = w" +
                 std::to_string(j) + ";").c_str()
              : "");
    }
    o("  __syncthreads();");

    int tl_of_pos[64];
    for (int p = 0; p < 64; ++p) tl_of_pos[p] = -1;
    for (int t = 0; t < k; ++t) tl_of_pos[(int)sw.tb[t]] = t;

    for (int f = 0; f < sw.n_phases; ++f) {
        const DevPhase& ph = pass.phases[sw.phase_begin + f];
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
        o("  { // phase %d", f);
        o("    uint32_t s_t = 0;");
        for (int j = 0; j < k - R; ++j)
            o("    s_t ^= (0u - ((tid >> %d) & 1u)) & %uu;", j, swz_host(1u << ph.thr_tl[j], W));
        std::vector<uint32_t> offs(NR);
        for (int l = 0; l < NR; ++l) {
            uint32_t off = 0;
            for (int r = 0; r < R; ++r)
                if ((l >> r) & 1) off |= 1u << ph.reg_tl[r];
            offs[l] = swz_host(off, W);
        }
        for (int l = 0; l < NR; ++l) {
            if (bwd)
                o("    V x%d = tile[s_t ^ %uu]; V y%d = tile2[s_t ^ %uu];", l, offs[l], l, offs[l]);
            else
                o("    V x%d = tile[s_t ^ %uu];", l, offs[l]);
        }
        std::vector<int> phys(NR);
        for (int l = 0; l < NR; ++l) phys[l] = l;
        std::vector<const char*> arrs = {"x"};
        if (bwd) arrs.push_back("y");
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
        for (int oi = ph.op_begin; oi < ph.op_end; ++oi) {
            const DevOp& op = pass.ops[oi];
            switch (op.kind) {
                case DK_G1: case DK_R1: case DK_RX: {
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
                case DK_X1:
                    rename(op.rb0, -1);
                    break;
                case DK_CX:
                    if (op.rb1 >= 0) {
                        rename(op.rb0, op.rb1);
                    } else {
                        BitSrc c = src(op.pos0);
                        o("    { const bool c = %s != 0u;", c.expr.c_str());
                        for (const char* A : arrs)
                            for (auto pr : pairs(op.rb0)) o("      jcswap(%s%d, %s%d, c);", A, pr.first, A, pr.second);
                        o("    }");
                    }
                    break;
                case DK_D1: {
                    o("    { const V d0 = smat[%d], d1 = smat[%d];", op.moff, op.moff + 1);
                    BitSrc s0 = src(op.pos0);
                    if (s0.rb >= 0) {
                        for (const char* A : arrs)
                            for (int l = 0; l < NR; ++l)
                                o("      %s%d = cmul(%s%d, %s);", A, phys[l], A, phys[l], ((l >> s0.rb) & 1) ? "d1" : "d0");
                    } else {
                        o("      const V d = %s ? d1 : d0;", s0.expr.c_str());
                        for (const char* A : arrs)
                            for (int l = 0; l < NR; ++l) o("      %s%d = cmul(%s%d, d);", A, phys[l], A, phys[l]);
                    }
                    o("    }");
                    break;
                }
                case DK_D2: {
                    o("    { const V d00 = smat[%d], d01 = smat[%d], d10 = smat[%d], d11 = smat[%d];", op.moff,
                      op.moff + 1, op.moff + 2, op.moff + 3);
                    BitSrc s0 = src(op.pos0), s1 = src(op.pos1);
                    if (s0.rb < 0 && s1.rb < 0) {
                        o("      const V d = %s ? (%s ? d11 : d10) : (%s ? d01 : d00);", s0.expr.c_str(),
                          s1.expr.c_str(), s1.expr.c_str());
                        for (const char* A : arrs)
                            for (int l = 0; l < NR; ++l) o("      %s%d = cmul(%s%d, d);", A, phys[l], A, phys[l]);
                    } else if (s0.rb >= 0 && s1.rb >= 0) {
                        const char* dn[4] = {"d00", "d01", "d10", "d11"};
                        for (const char* A : arrs)
                            for (int l = 0; l < NR; ++l)
                                o("      %s%d = cmul(%s%d, %s);", A, phys[l], A, phys[l],
                                  dn[(((l >> s0.rb) & 1) << 1) | ((l >> s1.rb) & 1)]);
                    } else if (s0.rb >= 0) {  // wire 1 runtime
                        o("      const V e0 = %s ? d01 : d00, e1 = %s ? d11 : d10;", s1.expr.c_str(), s1.expr.c_str());
                        for (const char* A : arrs)
                            for (int l = 0; l < NR; ++l)
                                o("      %s%d = cmul(%s%d, %s);", A, phys[l], A, phys[l], ((l >> s0.rb) & 1) ? "e1" : "e0");
                    } else {  // wire 0 runtime
                        o("      const V e0 = %s ? d10 : d00, e1 = %s ? d11 : d01;", s0.expr.c_str(), s0.expr.c_str());
                        for (const char* A : arrs)
                            for (int l = 0; l < NR; ++l)
                                o("      %s%d = cmul(%s%d, %s);", A, phys[l], A, phys[l], ((l >> s1.rb) & 1) ? "e1" : "e0");
                    }
                    o("    }");
                    break;
                }
                case DK_G2: {
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
                case DK_TX: case DK_TY: case DK_TZ: case DK_TZZ: {
                    o("    { RT s = 0;");
                    if (op.kind == DK_TX) {
                        for (auto pr : pairs(op.rb0))
                            o("      s += imcv(y%d, x%d) + imcv(y%d, x%d);", pr.first, pr.second, pr.second, pr.first);
                    } else if (op.kind == DK_TY) {
                        for (auto pr : pairs(op.rb0))
                            o("      s += recv(y%d, x%d) - recv(y%d, x%d);", pr.second, pr.first, pr.first, pr.second);
                    } else {
                        BitSrc s0 = src(op.pos0);
                        BitSrc s1 = op.kind == DK_TZZ ? src(op.pos1) : BitSrc{};
                        for (int l = 0; l < NR; ++l) {
                            int sg = 0;
                            if (s0.rb >= 0) sg ^= (l >> s0.rb) & 1;
                            if (op.kind == DK_TZZ && s1.rb >= 0) sg ^= (l >> s1.rb) & 1;
                            o("      s %s= imcv(y%d, x%d);", sg ? "-" : "+", phys[l], phys[l]);
                        }
                        std::string rt;
                        if (s0.rb < 0) rt = s0.expr;
                        if (op.kind == DK_TZZ && s1.rb < 0) rt = rt.empty() ? s1.expr : "(" + rt + " ^ " + s1.expr + ")";
                        if (!rt.empty()) o("      if (%s) s = -s;", rt.c_str());
                    }
                    o("      tap_store<RT>(s, stap, %d, %d, %d); }", op.tap, nwarps, T);
                    break;
                }
                default:
                    break;
            }
        }
        for (int l = 0; l < NR; ++l) {
            if (bwd)
                o("    tile[s_t ^ %uu] = x%d; tile2[s_t ^ %uu] = y%d;", offs[l], phys[l], offs[l], phys[l]);
            else
                o("    tile[s_t ^ %uu] = x%d;", offs[l], phys[l]);
        }
        o("    __syncthreads();");
        o("  }");
    }
    for (int j = 0; j < NR; ++j) {
        if (bwd)
            o("  v%d = tile[swz<%d>(tid + %uu)]; w%d = tile2[swz<%d>(tid + %uu)];", j, W, (unsigned)(T * j), j, W,
              (unsigned)(T * j));
        else
            o("  v%d = tile[swz<%d>(tid + %uu)];", j, W, (unsigned)(T * j));
    }
    for (int j = 0; j < NR; ++j) {
        if (bwd)
            o("  st[g_ld | %uu] = v%d; lm[g_ld | %uu] = w%d;", joff[j], j, joff[j], j);
        else
            o("  st[g_ld | %uu] = v%d;", joff[j], j);
    }
    if (bwd && sw.n_taps > 0) {
        o("  for (int t = (int)tid; t < %d; t += %d) {", sw.n_taps, T);
        o("    double s = 0;");
        o("    for (int w = 0; w < %d; ++w) s += stap[t * %d + w];", nwarps, nwarps);
        o("    a.tap_part[((size_t)b * a.n_taps_total + %d + t) * gridDim.x + tile_id] = s;", sw.tap_begin);
        o("  }");
    }
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

bool compile_one(const std::string& src, std::string& cubin, std::string& err) {
    static const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DQF_JIT=1"};
    nvrtcProgram prog = nullptr;
    if (g_nvrtc.create(&prog, src.c_str(), "qf_sweep.cu", 0, nullptr, nullptr) != 0) {
        err = "nvrtcCreateProgram failed";
        return false;
    }
    int rc = g_nvrtc.compile(prog, 4, opts);
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

struct Job {
    const ProgramPlan* P;
    const PassPlan* pass;
    int si;
    bool bwd;
    std::string cubin, err;
    bool from_cache = false;
};

}  // namespace

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

bool jit_build(const ProgramPlan& P, JitPass& fwd, JitPass& bwd, JitStats& st) {
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
    std::atomic<size_t> next{0};
    auto worker = [&] {
        for (;;) {
            size_t j = next.fetch_add(1);
            if (j >= jobs.size()) return;
            Job& jb = jobs[j];
            const std::string src = jit_source(*jb.P, *jb.pass, jb.si, jb.bwd);
            char key[64];
            snprintf(key, sizeof key, "%016llx_%d_%d", (unsigned long long)fnv1a(src), maj, min);
            const std::string path = dir + "/" + key + ".cubin";
            if (read_file(path, jb.cubin)) {
                jb.from_cache = true;
                continue;
            }
            if (!compile_one(src, jb.cubin, jb.err)) continue;
            const std::string tmp = path + ".tmp" + std::to_string(getpid()) + "_" + std::to_string(j);
            {
                std::ofstream f(tmp, std::ios::binary);
                f.write(jb.cubin.data(), (std::streamsize)jb.cubin.size());
            }
            rename(tmp.c_str(), path.c_str());
        }
    };
    unsigned nthr = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("QF_JIT_THREADS")) nthr = (unsigned)std::max(1, atoi(e));
    nthr = std::max(1u, std::min<unsigned>(nthr, (unsigned)jobs.size()));
    std::vector<std::thread> pool;
    for (unsigned i = 0; i < nthr; ++i) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    fwd.sweeps.assign(P.fwd.sweeps.size(), {});
    bwd.sweeps.assign(P.bwd.sweeps.size(), {});
    for (auto& jb : jobs) {
        if (!jb.err.empty()) {
            st.error = jb.err;
            return false;
        }
        cudaLibrary_t lib;
        cudaError_t e = cudaLibraryLoadData(&lib, jb.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
        if (e != cudaSuccess) {
            st.error = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
            return false;
        }
        cudaKernel_t kern;
        e = cudaLibraryGetKernel(&kern, lib, "qf_sweep");
        if (e != cudaSuccess) {
            st.error = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
            return false;
        }
        JitKernel jk;
        jk.kernel = (void*)kern;
        const DevSweep& sw = jb.pass->sweeps[jb.si];
        jk.threads = 1 << (sw.k - sw.R);
        jk.smem = jit_smem_bytes(P, *jb.pass, jb.si, jb.bwd);
        if (jk.smem > 48 * 1024) {
            e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jk.smem);
            if (e != cudaSuccess) {
                st.error = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
                return false;
            }
        }
        (jb.bwd ? bwd : fwd).sweeps[jb.si] = jk;
        if (jb.from_cache) st.cached++;
        else st.compiled++;
    }
    fwd.ok = bwd.ok = true;
    st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return true;
}

int jit_launch(const JitKernel& k, const SweepArgs& a, int tiles, int batch, void* stream) {
    void* args[] = {const_cast<SweepArgs*>(&a)};
    cudaError_t e = cudaLaunchKernel((const void*)k.kernel, dim3(tiles, batch), dim3(k.threads), args, k.smem,
                                     (cudaStream_t)stream);
    return (int)e;
}

}  // namespace qfb
