// capi.cpp -- the C-ABI (include/qforge_b200.h): contexts, compiled programs and
// observables, chunked batch evaluation, NCCL sharding.
//
// Evaluation of one batch chunk (all on the context stream, no host sync):
//   forward sweeps (fused tile kernels) -> H|psi> + energy partials ->
//   adjoint sweeps with gradient taps -> fixed-order reductions.
// The reference evaluates 1 + 2P full energies per gradient
// (src/variational.cpp:54-81); this evaluates one forward and one adjoint pass.
#include <array>
#include <atomic>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <chrono>
#include <complex>
#include <thread>

#include <cublas_v2.h>
#include <cusolverDn.h>

#include "../../include/qforge_b200.h"
#include "../../include/qforge/rng.hpp"
#include "kernels.cuh"
#include "jit.hpp"
#include "plan.hpp"

using namespace qfb;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

static std::string launch_detail(const char* call) {
    return std::strstr(call, "jit_launch") ? " [" + qfb::jit_last_launch_detail() + "]" : std::string();
}

#define QF_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_err(QF_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                         " at " #call + launch_detail(#call));            \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct LocalBuf : DevBuf {  // function-scoped device scratch
    ~LocalBuf() { release(); }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMallocHost(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

template <typename T> cudaError_t upload(DevBuf& b, const std::vector<T>& v, cudaStream_t s) {
    size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
    cudaError_t e = b.reserve(bytes);
    if (e != cudaSuccess) return e;
    if (!v.empty()) e = cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    return e;
}

// ---- NCCL, loaded lazily (torch already ships libnccl.so.2) ----
typedef struct { char internal[128]; } NcclId;
typedef void* NcclComm;
struct NcclApi {
    void* h = nullptr;
    int (*getUniqueId)(NcclId*) = nullptr;
    int (*commInitRank)(NcclComm*, int, NcclId, int) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    int (*commDestroy)(NcclComm) = nullptr;
    const char* (*errStr)(int) = nullptr;
    bool load(std::string& why) {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so",
                               "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
        for (const char* nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            why = "cannot load libnccl.so.2";
            return false;
        }
        getUniqueId = (int (*)(NcclId*))dlsym(h, "ncclGetUniqueId");
        commInitRank = (int (*)(NcclComm*, int, NcclId, int))dlsym(h, "ncclCommInitRank");
        allReduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllReduce");
        commDestroy = (int (*)(NcclComm))dlsym(h, "ncclCommDestroy");
        errStr = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
        if (!getUniqueId || !commInitRank || !allReduce || !commDestroy || !errStr) {
            why = "libnccl.so.2 lacks required symbols";
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;
std::mutex g_nccl_mu;
constexpr int kNcclFloat64 = 8, kNcclSum = 0;

}  // namespace

struct qf_observable;

struct DevPass {
    DevBuf phases, ops;
};

struct qf_program {
    qf_ctx* ctx = nullptr;
    ProgramPlan plan;
    DevBuf gates, cmats;
    DevPass fwd, bwd;
    DevBuf slot_ptr, slot_taps, slot_coef;
    DevBuf goff_fwd, goff_bwd;  // per op: offset of its matrix in the per-state table (-1: none)
    DevBuf init;  // optional initial state (RT)
    bool has_init = false;
    // NVRTC-specialised sweep kernels (jit.hpp); the AOT interpreter is the fallback
    bool use_jit = false;
    JitPass jf, jb;
    JitStats jst;
};

struct ObsDev {
    ObservablePlan plan;
    DevBuf groups, terms;
    bool ready = false;
    JitKernel hj;       // specialised H|psi> kernel (jit.hpp)
    int hj_state = 0;   // 0 not built, 1 ready, -1 unavailable (AOT hpsi_kernel)
};

struct qf_observable {
    qf_ctx* ctx = nullptr;
    int n = 0;
    std::vector<int8_t> codes;
    std::vector<double> w_re, w_im;
    ObsDev dev[2];         // per precision (tile bits differ)
    bool term_shard = false;
    int shard_world = 0;   // term-sharded sub-plan cache key
    ObsDev shard_dev[2];
    uint64_t uid = 0;      // identity for the context's COO offset cache
};

struct qf_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    size_t budget = 0;
    DevBuf psi, lam, tap_part, tapsum, epart, thetas, out, zero_init, gmat;
    DevBuf coo_off, coo_scratch, coo_groups, coo_terms, coo_nodes, coo_rows, coo_cols, coo_vals;
    uint64_t coo_uid = 0;  // observable whose groups/terms/offsets coo_* currently hold (0: none)
    std::map<std::pair<int, int>, qf_program*> basis_progs;  // (n, precision) -> per-qubit basis rotation program
    int coo_n_groups = 0, coo_n_events = 0, coo_n_terms = 0;
    int64_t coo_total = 0;
    HostBuf pin;
    // NCCL
    NcclComm comm = nullptr;
    int rank = 0, world = 1;
    // stats (accumulated until qf_ctx_reset_stats); timing uses event pairs
    // recorded on the context stream and resolved lazily (no mid-call syncs)
    bool timing = false;
    long long launches = 0;
    long long class_launches[4] = {0, 0, 0, 0};
    double ms[4] = {0, 0, 0, 0};
    double bytes[4] = {0, 0, 0, 0};
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<size_t, int>> pending;  // (start event index, class); end = start + 1
};

namespace {

int ensure_obs_dev(qf_observable* o, int prec, int kh, ObsDev& d, int t_begin, int t_end) {
    if (d.ready && d.plan.kh == kh) return QF_OK;
    std::string e = build_observable_plan(o->n, t_end - t_begin, o->codes.data() + (size_t)t_begin * o->n,
                                          o->w_re.data() + t_begin, o->w_im.data() + t_begin, kh, d.plan);
    if (!e.empty()) return set_err(QF_EINVAL, e);
    cudaStream_t s = o->ctx->stream;
    QF_CUDA(upload(d.groups, d.plan.groups, s));
    QF_CUDA(upload(d.terms, d.plan.terms, s));
    d.ready = true;
    d.hj_state = 0;  // plan (re)built: the specialised H|psi> kernel follows it
    (void)prec;
    return QF_OK;
}

size_t vsize(int prec) { return prec == QF_C128 ? 16 : 8; }

void resolve_events(qf_ctx* ctx) {
    if (ctx->pending.empty()) {
        ctx->ev_used = 0;
        return;
    }
    cudaStreamSynchronize(ctx->stream);
    for (auto& pr : ctx->pending) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ctx->ev_pool[pr.first], ctx->ev_pool[pr.first + 1]);
        ctx->ms[pr.second] += ms;
    }
    ctx->pending.clear();
    ctx->ev_used = 0;
}

// records an event on s; start/end pairs are consecutive in the pool
size_t record_event(qf_ctx* ctx, cudaStream_t s) {
    if (ctx->ev_used >= 4096 && ctx->ev_used % 2 == 0) resolve_events(ctx);
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
    }
    cudaEventRecord(ctx->ev_pool[ctx->ev_used], s);
    return ctx->ev_used++;
}

// one chunk: [b0, b0 + bc) of d_thetas rows
int eval_chunk(qf_ctx* ctx, qf_program* prog, ObsDev* od, int b0, int bc, const double* d_thetas,
               double* d_E, double* d_Eim, double* d_G, ObsDev* od_im) {
    const ProgramPlan& P = prog->plan;
    const int n = P.n, prec = P.prec;
    const size_t N = size_t(1) << n;
    const size_t vs = vsize(prec);
    cudaStream_t s = ctx->stream;
    const bool grads = d_G != nullptr;
    const int P_ = P.n_params;
    size_t ev_start[4] = {0, 0, 0, 0};
    auto tick = [&](int i) {
        if (ctx->timing) ev_start[i / 2] = record_event(ctx, s);
    };
    auto tock = [&](int i, int cls) {
        if (ctx->timing) {
            record_event(ctx, s);
            ctx->pending.push_back({ev_start[i / 2], cls});
        }
    };

    // --- forward ---
    tick(0);
    SweepArgs sa{};
    sa.psi = ctx->psi.p;
    sa.lam = ctx->lam.p;
    sa.theta = d_thetas;
    sa.P = P_;
    sa.n = n;
    sa.batch_offset = b0;
    sa.gates = (const DevGate*)prog->gates.p;
    sa.cmats = (const double*)prog->cmats.p;
    sa.gmat = ctx->gmat.p;
    sa.gmat_stride = P.fwd.total_mat + P.bwd.total_mat;
    sa.gmat_pass_base = 0;
    QF_CUDA(launch_mats(prec, false, (const DevOp*)prog->fwd.ops.p, (const int*)prog->goff_fwd.p,
                        (int)P.fwd.ops.size(), sa.gates, sa.cmats, d_thetas, P_, b0, ctx->gmat.p, sa.gmat_stride, 0,
                        bc, s));
    ctx->launches++;
    if (grads) {
        QF_CUDA(launch_mats(prec, true, (const DevOp*)prog->bwd.ops.p, (const int*)prog->goff_bwd.p,
                            (int)P.bwd.ops.size(), sa.gates, sa.cmats, d_thetas, P_, b0, ctx->gmat.p,
                            sa.gmat_stride, P.fwd.total_mat, bc, s));
        ctx->launches++;
    }
    const bool first_from_zero = !prog->has_init && !P.fwd.sweeps.empty();
    if (prog->has_init) {
        QF_CUDA(launch_init_state(prec, ctx->psi.p, prog->init.p, n, bc, s));
        ctx->launches++;
    } else if (P.fwd.sweeps.empty()) {
        QF_CUDA(launch_init_state(prec, ctx->psi.p, ctx->zero_init.p, n, bc, s));
        ctx->launches++;
    }
    sa.phases = (const DevPhase*)prog->fwd.phases.p;
    sa.ops = (const DevOp*)prog->fwd.ops.p;
    for (size_t i = 0; i < P.fwd.sweeps.size(); ++i) {
        sa.sw = P.fwd.sweeps[i];
        sa.from_zero = (i == 0 && first_from_zero) ? 1 : 0;
        if (prog->use_jit)
            QF_CUDA((cudaError_t)jit_launch(prog->jf.sweeps[i], sa, 1 << (n - sa.sw.k), bc, s));
        else
            QF_CUDA(launch_sweep(prec, false, sa, bc, P.fwd.max_mat, 0, s));
        ctx->launches++;
        ctx->class_launches[0]++;
        ctx->bytes[0] += (double)bc * N * vs * (sa.from_zero ? 1 : 2);
    }
    if (!prog->has_init && P.fwd.sweeps.empty()) ctx->bytes[0] += (double)bc * N * vs;
    tock(0, 0);

    // --- H|psi>, energy ---
    tick(2);
    const int kh = od->plan.kh;
    const int tiles_h = 1 << (n - kh);
    HArgs ha{};
    ha.psi = ctx->psi.p;
    ha.lam = ctx->lam.p;
    ha.n = n;
    ha.kh = kh;
    ha.groups = (const DevGroup*)od->groups.p;
    ha.n_groups = (int)od->plan.groups.size();
    ha.terms = (const DevTerm*)od->terms.p;
    ha.write_lam = grads ? 1 : 0;
    ha.use_imag = 0;
    ha.epart = (double*)ctx->epart.p;
    if (prog->use_jit && od->hj_state == 0 && !(std::getenv("QF_JIT_HPSI") && std::getenv("QF_JIT_HPSI")[0] == '0')) {
        std::string err;
        od->hj_state = ((int)od->plan.terms.size() <= kJitHpsiMaxTerms && jit_build_hpsi(od->plan, prec, od->hj, err))
                           ? 1 : -1;
    }
    if (od->hj_state == 1)
        QF_CUDA((cudaError_t)jit_launch_hpsi(od->hj, ha, tiles_h, bc, s));
    else
        QF_CUDA(launch_hpsi(prec, ha, bc, s));
    ctx->launches++;
    ctx->class_launches[1]++;
    ctx->bytes[1] += (double)bc * N * vs * (ha.n_groups + (grads ? 1 : 0));
    ReduceArgs ra{};
    ra.part = (const double*)ctx->epart.p;
    ra.count = 1;
    ra.tiles = tiles_h;
    ra.out = d_E + b0;
    QF_CUDA(launch_reduce(ra, bc, s));
    ctx->launches++;
    if (d_Eim && od_im) {
        HArgs hi = ha;
        hi.groups = (const DevGroup*)od_im->groups.p;
        hi.n_groups = (int)od_im->plan.groups.size();
        hi.terms = (const DevTerm*)od_im->terms.p;
        hi.write_lam = 0;
        hi.use_imag = 1;
        QF_CUDA(launch_hpsi(prec, hi, bc, s));
        ra.out = d_Eim + b0;
        QF_CUDA(launch_reduce(ra, bc, s));
        ctx->launches += 2;
    }
    tock(2, 1);

    // --- adjoint ---
    if (grads) {
        tick(4);
        const int nt = P.bwd.n_taps;
        const int tiles_b = 1 << (n - P.bwd.k);
        sa.phases = (const DevPhase*)prog->bwd.phases.p;
        sa.ops = (const DevOp*)prog->bwd.ops.p;
        sa.from_zero = 0;
        sa.tap_part = (double*)ctx->tap_part.p;
        sa.n_taps_total = nt;
        sa.gmat_pass_base = P.fwd.total_mat;
        for (size_t i = 0; i < P.bwd.sweeps.size(); ++i) {
            sa.sw = P.bwd.sweeps[i];
            if (prog->use_jit)
                QF_CUDA((cudaError_t)jit_launch(prog->jb.sweeps[i], sa, 1 << (n - sa.sw.k), bc, s));
            else
                QF_CUDA(launch_sweep(prec, true, sa, bc, P.bwd.max_mat, P.bwd.max_taps, s));
            ctx->launches++;
            ctx->class_launches[2]++;
            ctx->bytes[2] += (double)bc * N * vs * 4;
        }
        tock(4, 2);
        tick(6);
        if (nt > 0) {
            ReduceArgs rt{};
            rt.part = (const double*)ctx->tap_part.p;
            rt.count = nt;
            rt.tiles = tiles_b;
            rt.out = (double*)ctx->tapsum.p;
            QF_CUDA(launch_reduce(rt, bc, s));
            ctx->launches++;
        }
        QF_CUDA(launch_gather_grads((const double*)ctx->tapsum.p, nt, (const int*)prog->slot_ptr.p,
                                    (const int*)prog->slot_taps.p, (const double*)prog->slot_coef.p,
                                    P_, bc, d_G + (size_t)b0 * P_, s));
        ctx->launches++;
        tock(6, 3);
    }
    return QF_OK;
}

// Evaluate rows [0, batch) of device thetas into device outputs (chunked).
int eval_device(qf_ctx* ctx, qf_program* prog, qf_observable* obs, int batch, const double* d_thetas,
                double* d_E, double* d_Eim, double* d_G, bool term_shard) {
    const ProgramPlan& P = prog->plan;
    if (obs->n != P.n) return set_err(QF_EINVAL, "expectation_pauli: size mismatch");
    if (d_G && !P.adjoint_ok) return set_err(QF_EINVAL, P.adjoint_error);
    const int prec = P.prec, n = P.n;
    const Geometry geo = geometry(prec, n);
    ObsDev* od = &obs->dev[prec];
    int rc;
    if (term_shard && ctx->comm) {
        const int T = (int)obs->w_re.size();
        const int t0 = (int)((long long)T * ctx->rank / ctx->world);
        const int t1 = (int)((long long)T * (ctx->rank + 1) / ctx->world);
        if (obs->shard_world != ctx->world) {
            obs->shard_dev[0].ready = obs->shard_dev[1].ready = false;
            obs->shard_world = ctx->world;
        }
        od = &obs->shard_dev[prec];
        rc = ensure_obs_dev(obs, prec, geo.kh, *od, t0, t1);
    } else {
        rc = ensure_obs_dev(obs, prec, geo.kh, *od, 0, (int)obs->w_re.size());
    }
    if (rc) return rc;
    ObsDev* od_im = (d_Eim && od->plan.has_imag) ? od : nullptr;
    if (d_Eim && !od_im) QF_CUDA(cudaMemsetAsync(d_Eim, 0, sizeof(double) * batch, ctx->stream));

    const size_t N = size_t(1) << n;
    const size_t vs = vsize(prec);
    const bool grads = d_G != nullptr;
    const int nt = P.bwd.n_taps;
    const size_t tiles_b = size_t(1) << (n - P.bwd.k);
    const size_t tiles_h = size_t(1) << (n - geo.kh);
    const size_t per_entry = N * vs * (grads ? 2 : 1) + (grads ? (size_t)nt * tiles_b * 8 + (size_t)nt * 8 : 0) +
                             tiles_h * 8 + (size_t)(P.fwd.total_mat + P.bwd.total_mat) * vs;
    size_t budget = ctx->budget;
    if (!budget) {
        size_t fr = 0, tot = 0;
        QF_CUDA(cudaMemGetInfo(&fr, &tot));
        budget = (size_t)(0.6 * (double)(fr + ctx->psi.cap + ctx->lam.cap + ctx->tap_part.cap));
    }
    long long bc = std::max<long long>(1, (long long)(budget / per_entry));
    bc = std::min<long long>(bc, batch);
    bc = std::min<long long>(bc, 65535);
    // even chunks
    const long long nchunks = (batch + bc - 1) / bc;
    bc = (batch + nchunks - 1) / nchunks;
    QF_CUDA(ctx->psi.reserve(bc * N * vs));
    if (grads) {
        QF_CUDA(ctx->lam.reserve(bc * N * vs));
        QF_CUDA(ctx->tap_part.reserve(std::max<size_t>(16, bc * (size_t)nt * tiles_b * 8)));
        QF_CUDA(ctx->tapsum.reserve(std::max<size_t>(16, bc * (size_t)nt * 8)));
    }
    QF_CUDA(ctx->epart.reserve(bc * tiles_h * 8));
    QF_CUDA(ctx->gmat.reserve(std::max<size_t>(16, bc * (size_t)(P.fwd.total_mat + P.bwd.total_mat) * vs)));
    if (!prog->has_init && P.fwd.sweeps.empty()) {
        if (ctx->zero_init.cap < N * vs) {
            QF_CUDA(ctx->zero_init.reserve(N * vs));
        }
        QF_CUDA(cudaMemsetAsync(ctx->zero_init.p, 0, N * vs, ctx->stream));
        if (prec == QF_C128) {
            double one[2] = {1.0, 0.0};
            QF_CUDA(cudaMemcpyAsync(ctx->zero_init.p, one, 16, cudaMemcpyHostToDevice, ctx->stream));
        } else {
            float one[2] = {1.0f, 0.0f};
            QF_CUDA(cudaMemcpyAsync(ctx->zero_init.p, one, 8, cudaMemcpyHostToDevice, ctx->stream));
        }
        QF_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    for (long long b0 = 0; b0 < batch; b0 += bc) {
        const int c = (int)std::min<long long>(bc, batch - b0);
        rc = eval_chunk(ctx, prog, od, (int)b0, c, d_thetas, d_E, d_Eim, d_G, od_im);
        if (rc) return rc;
    }
    return QF_OK;
}

int check_thetas(const qf_program* prog, int batch, const double* thetas) {
    const ProgramPlan& P = prog->plan;
    for (const auto& gi : P.gates) {
        if (gi.g.slot < 0) continue;
        for (int b = 0; b < batch; ++b) {
            const double p = gi.g.coef * thetas[(size_t)b * P.n_params + gi.g.slot] + gi.g.offset;
            if (!std::isfinite(p)) return set_err(QF_EINVAL, "Circuit: non-finite parameter");
        }
    }
    return QF_OK;
}

// ------------------------------------------------------------------ trajectories
// haar_su4 (reference circuit.cpp:472-489): QR of a complex Gaussian 4x4 with the
// phases of R's diagonal moved into Q (the unique QR with positive diagonal,
// computed here by modified Gram-Schmidt), then Q *= det(Q)^(-1/4).  Entries are
// drawn as cplx(rng.normal(), rng.normal()); gcc evaluates those arguments right
// to left, so the imaginary part is drawn first (pinned by
// tests/golden/rng_known_answers.txt through the same convention).
using cd = std::complex<double>;
void haar_su4(qforge::RngStream& rng, cd q[4][4]) {
    cd g[4][4];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            const double im = rng.normal();
            const double re = rng.normal();
            g[r][c] = cd(re, im);
        }
    for (int j = 0; j < 4; ++j) {
        cd v[4] = {g[0][j], g[1][j], g[2][j], g[3][j]};
        for (int i = 0; i < j; ++i) {
            cd d = 0;
            for (int r = 0; r < 4; ++r) d += std::conj(q[r][i]) * v[r];
            for (int r = 0; r < 4; ++r) v[r] -= d * q[r][i];
        }
        double nr = 0;
        for (int r = 0; r < 4; ++r) nr += std::norm(v[r]);
        nr = std::sqrt(nr);
        for (int r = 0; r < 4; ++r) q[r][j] = v[r] / nr;
    }
    // det by Gaussian elimination with partial pivoting
    cd a[4][4];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) a[r][c] = q[r][c];
    cd det = 1.0;
    for (int c = 0; c < 4; ++c) {
        int piv = c;
        for (int r = c + 1; r < 4; ++r)
            if (std::abs(a[r][c]) > std::abs(a[piv][c])) piv = r;
        if (piv != c) {
            for (int k = 0; k < 4; ++k) std::swap(a[piv][k], a[c][k]);
            det = -det;
        }
        det *= a[c][c];
        for (int r = c + 1; r < 4; ++r) {
            const cd f = a[r][c] / a[c][c];
            for (int k = c; k < 4; ++k) a[r][k] -= f * a[c][k];
        }
    }
    const cd ph = std::polar(1.0, -std::arg(det) / 4.0);
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) q[r][c] *= ph;
}

// gate_matrix (reference circuit.cpp:202-302) on the host for the noise
// trajectories: D x D row-major (wires[0] most significant), angle = op.offset
int host_gate_matrix(const qf_op& o, const double* mats, int n_mats, int& D, cd m[16]) {
    for (int i = 0; i < 16; ++i) m[i] = 0.0;
    const double t = o.offset, c = std::cos(0.5 * t), sn = std::sin(0.5 * t), h = std::sqrt(0.5);
    const cd I(0.0, 1.0);
    D = 2;
    switch (o.kind) {
        case QF_H: m[0] = h; m[1] = h; m[2] = h; m[3] = -h; break;
        case QF_X: m[1] = 1; m[2] = 1; break;
        case QF_Y: m[1] = -I; m[2] = I; break;
        case QF_Z: m[0] = 1; m[3] = -1; break;
        case QF_S: m[0] = 1; m[3] = I; break;
        case QF_RX: m[0] = c; m[1] = -I * sn; m[2] = -I * sn; m[3] = c; break;
        case QF_RY: m[0] = c; m[1] = -sn; m[2] = sn; m[3] = c; break;
        case QF_RZ: m[0] = std::polar(1.0, -0.5 * t); m[3] = std::polar(1.0, 0.5 * t); break;
        case QF_RZZ:
            D = 4;
            m[0] = m[15] = std::polar(1.0, -0.5 * t);
            m[5] = m[10] = std::polar(1.0, 0.5 * t);
            break;
        case QF_CX: D = 4; m[0] = m[5] = m[11] = m[14] = 1; break;
        case QF_CZ: D = 4; m[0] = m[5] = m[10] = 1; m[15] = -1; break;
        case QF_SU4: case QF_UNITARY: {
            if (o.mat < 0 || o.mat >= n_mats || !mats) return set_err(QF_EINVAL, "program: missing gate matrix");
            D = o.q1 >= 0 ? 4 : 2;
            const double* src = mats + 32 * (size_t)o.mat;
            for (int r = 0; r < D; ++r)
                for (int cc = 0; cc < D; ++cc) m[r * D + cc] = cd(src[(r * 4 + cc) * 2], src[(r * 4 + cc) * 2 + 1]);
            break;
        }
        default: return set_err(QF_EINVAL, "gate_matrix: qudit gates are not supported on the qubit device path");
    }
    return QF_OK;
}

// cuBLAS / cuSOLVER, loaded at run time (only the trajectory entropy needs them)
struct LinAlg {
    void *hb = nullptr, *hs = nullptr;
    cublasHandle_t cb = nullptr;
    cusolverDnHandle_t cs = nullptr;
    decltype(&cublasCreate_v2) bcreate = nullptr;
    decltype(&cublasSetStream_v2) bstream = nullptr;
    decltype(&cublasZherk_v2) zherk = nullptr;
    decltype(&cusolverDnCreate) screate = nullptr;
    decltype(&cusolverDnSetStream) sstream = nullptr;
    decltype(&cusolverDnZheevd_bufferSize) zheevd_ws = nullptr;
    decltype(&cusolverDnZheevd) zheevd = nullptr;
    std::string err;
    bool load() {
        if (cb && cs) return true;
        const char* bl[] = {"libcublas.so.12", "libcublas.so", "/usr/local/cuda/lib64/libcublas.so.12",
                            "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cublas/lib/libcublas.so.12"};
        const char* sl[] = {"libcusolver.so.11", "libcusolver.so", "/usr/local/cuda/lib64/libcusolver.so.11",
                            "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cusolver/lib/libcusolver.so.11"};
        for (const char* nm : bl)
            if ((hb = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
        for (const char* nm : sl)
            if ((hs = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
        if (!hb || !hs) {
            err = "cuBLAS / cuSOLVER unavailable (libcublas.so.12 / libcusolver.so.11)";
            return false;
        }
        bcreate = (decltype(bcreate))dlsym(hb, "cublasCreate_v2");
        bstream = (decltype(bstream))dlsym(hb, "cublasSetStream_v2");
        zherk = (decltype(zherk))dlsym(hb, "cublasZherk_v2");
        screate = (decltype(screate))dlsym(hs, "cusolverDnCreate");
        sstream = (decltype(sstream))dlsym(hs, "cusolverDnSetStream");
        zheevd_ws = (decltype(zheevd_ws))dlsym(hs, "cusolverDnZheevd_bufferSize");
        zheevd = (decltype(zheevd))dlsym(hs, "cusolverDnZheevd");
        if (!bcreate || !bstream || !zherk || !screate || !sstream || !zheevd_ws || !zheevd) {
            err = "cuBLAS / cuSOLVER lack required symbols";
            return false;
        }
        if (bcreate(&cb) != CUBLAS_STATUS_SUCCESS || screate(&cs) != CUSOLVER_STATUS_SUCCESS) {
            err = "cuBLAS / cuSOLVER handle creation failed";
            return false;
        }
        return true;
    }
};
LinAlg g_linalg;
std::mutex g_linalg_mu;

// One ZHEEVD of a 1024 x 1024 matrix is latency bound (~12 ms on one stream);
// spectra run concurrently on kEigLanes host threads, each with its own stream,
// cuBLAS / cuSOLVER handles and scratch.
constexpr int kEigLanes = 8;
struct EigLane {
    int device = -1;
    cudaStream_t st = nullptr;
    cublasHandle_t cb = nullptr;
    cusolverDnHandle_t cs = nullptr;
    DevBuf conv, rho, work, info;
    int64_t dk = 0;
    int lwork = 0;
};
EigLane g_lanes[kEigLanes];

int lane_setup(EigLane& L, const LinAlg& la, int device, int64_t dk, size_t N) {
    if (L.device != device) {
        if (L.st) {
            cudaStreamDestroy(L.st);
            L.st = nullptr;
        }
        L.cb = nullptr;
        L.cs = nullptr;
        L.device = device;
    }
    if (!L.st) QF_CUDA(cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking));
    if (!L.cb && la.bcreate(&L.cb) != CUBLAS_STATUS_SUCCESS) return set_err(QF_ERUNTIME, "cublasCreate failed");
    if (!L.cs && la.screate(&L.cs) != CUSOLVER_STATUS_SUCCESS) return set_err(QF_ERUNTIME, "cusolverDnCreate failed");
    if (la.bstream(L.cb, L.st) != CUBLAS_STATUS_SUCCESS || la.sstream(L.cs, L.st) != CUSOLVER_STATUS_SUCCESS)
        return set_err(QF_ERUNTIME, "cuBLAS / cuSOLVER stream binding failed");
    QF_CUDA(L.conv.reserve(N * 16));
    QF_CUDA(L.rho.reserve((size_t)dk * dk * 16));
    QF_CUDA(L.info.reserve(16));
    if (L.dk != dk) {
        if (la.zheevd_ws(L.cs, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, (int)dk,
                         (const cuDoubleComplex*)L.rho.p, (int)dk, nullptr, &L.lwork) != CUSOLVER_STATUS_SUCCESS)
            return set_err(QF_ERUNTIME, "cusolverDnZheevd_bufferSize failed");
        L.dk = dk;
    }
    QF_CUDA(L.work.reserve(std::max<size_t>(16, (size_t)L.lwork * 16)));
    return QF_OK;
}

}  // namespace

extern "C" {

int qf_abi_version(void) { return QF_ABI_VERSION; }
const char* qf_last_error(void) { return g_err.c_str(); }

int qf_ctx_create(int device, qf_ctx** out) {
    if (!out) return set_err(QF_EINVAL, "qf_ctx_create: null out");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return set_err(QF_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return set_err(QF_EINVAL, "qf_ctx_create: bad device index");
    QF_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    QF_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return set_err(QF_ECUDA, "qf_ctx_create: this build targets sm_100a (B200)");
    qf_ctx* c = new qf_ctx();
    c->device = device;
    QF_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c;
    return QF_OK;
}

int qf_ctx_destroy(qf_ctx* c) {
    if (!c) return QF_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->comm) g_nccl.commDestroy(c->comm);
    for (auto& kv : c->basis_progs) qf_program_destroy(kv.second);
    for (DevBuf* b : {&c->psi, &c->lam, &c->tap_part, &c->tapsum, &c->epart, &c->thetas, &c->out, &c->zero_init,
                      &c->gmat, &c->coo_off, &c->coo_scratch, &c->coo_groups, &c->coo_terms, &c->coo_nodes, &c->coo_rows,
                      &c->coo_cols, &c->coo_vals})
        b->release();
    c->pin.release();
    for (auto& ev : c->ev_pool) cudaEventDestroy(ev);
    cudaStreamDestroy(c->stream);
    delete c;
    return QF_OK;
}

int qf_ctx_set_memory_budget(qf_ctx* c, size_t bytes) {
    if (!c) return set_err(QF_EINVAL, "null context");
    c->budget = bytes;
    return QF_OK;
}

void* qf_ctx_stream(qf_ctx* c) { return c ? (void*)c->stream : nullptr; }

int qf_nccl_unique_id(uint8_t out[128]) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    std::string why;
    if (!g_nccl.load(why)) return set_err(QF_ENCCL, why);
    NcclId id;
    int r = g_nccl.getUniqueId(&id);
    if (r) return set_err(QF_ENCCL, std::string("ncclGetUniqueId: ") + g_nccl.errStr(r));
    std::memcpy(out, id.internal, 128);
    return QF_OK;
}

int qf_ctx_set_comm(qf_ctx* c, int rank, int world, const uint8_t unique_id[128]) {
    if (!c) return set_err(QF_EINVAL, "null context");
    if (world < 1 || rank < 0 || rank >= world) return set_err(QF_EINVAL, "qf_ctx_set_comm: bad rank/world");
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (c->comm) {
        g_nccl.commDestroy(c->comm);
        c->comm = nullptr;
    }
    c->rank = rank;
    c->world = world;
    bool zero_id = true;
    for (int i = 0; i < 128 && unique_id; ++i) zero_id &= unique_id[i] == 0;
    if (world == 1 && (zero_id || !unique_id)) return QF_OK;  // detach
    std::string why;
    if (!g_nccl.load(why)) return set_err(QF_ENCCL, why);
    QF_CUDA(cudaSetDevice(c->device));
    NcclId id;
    std::memcpy(id.internal, unique_id, 128);
    int r = g_nccl.commInitRank(&c->comm, world, id, rank);
    if (r) return set_err(QF_ENCCL, std::string("ncclCommInitRank: ") + g_nccl.errStr(r));
    return QF_OK;
}

int qf_program_create(qf_ctx* ctx, int n_qubits, int n_ops, const qf_op* ops, const double* mats,
                      int n_mats, int n_params, int precision, qf_program** out) {
    if (!ctx || !out) return set_err(QF_EINVAL, "qf_program_create: null argument");
    if (n_ops < 0 || (n_ops > 0 && !ops)) return set_err(QF_EINVAL, "qf_program_create: bad ops");
    std::vector<GateSpec> specs(n_ops);
    for (int i = 0; i < n_ops; ++i)
        specs[i] = GateSpec{ops[i].kind, ops[i].q0, ops[i].q1, ops[i].slot, ops[i].coef, ops[i].offset, ops[i].mat};
    qf_program* p = new qf_program();
    p->ctx = ctx;
    std::string e = build_program_plan(n_qubits, specs, mats, n_mats, n_params, precision, p->plan);
    if (!e.empty()) {
        delete p;
        return set_err(QF_EINVAL, e);
    }
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    std::vector<DevGate> dg(p->plan.gates.size());
    for (size_t i = 0; i < dg.size(); ++i) {
        const GateSpec& g = p->plan.gates[i].g;
        dg[i] = DevGate{g.kind, g.slot, g.coef, g.offset, g.mat, g.q0, g.q1};
    }
    auto fail = [&](cudaError_t ce) {
        delete p;
        return set_err(QF_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(ce));
    };
    cudaError_t ce;
    if ((ce = upload(p->gates, dg, s)) != cudaSuccess) return fail(ce);
    if ((ce = upload(p->cmats, p->plan.mats, s)) != cudaSuccess) return fail(ce);
    if ((ce = upload(p->fwd.phases, p->plan.fwd.phases, s)) != cudaSuccess) return fail(ce);
    if ((ce = upload(p->fwd.ops, p->plan.fwd.ops, s)) != cudaSuccess) return fail(ce);
    if ((ce = upload(p->bwd.phases, p->plan.bwd.phases, s)) != cudaSuccess) return fail(ce);
    if ((ce = upload(p->bwd.ops, p->plan.bwd.ops, s)) != cudaSuccess) return fail(ce);
    // slot -> taps CSR (taps summed in tap order: deterministic)
    const int P = n_params;
    std::vector<int> cnt(P + 1, 0), ptr(P + 1, 0), taps;
    std::vector<double> coef;
    for (const auto& t : p->plan.bwd.taps) cnt[t.slot]++;
    for (int i = 0; i < P; ++i) ptr[i + 1] = ptr[i] + cnt[i];
    taps.resize(ptr[P]);
    coef.resize(ptr[P]);
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (size_t t = 0; t < p->plan.bwd.taps.size(); ++t) {
        const auto& tp = p->plan.bwd.taps[t];
        taps[fill[tp.slot]] = (int)t;
        coef[fill[tp.slot]++] = tp.coef;
    }
    for (int pi = 0; pi < 2; ++pi) {
        const PassPlan& pp = pi ? p->plan.bwd : p->plan.fwd;
        std::vector<int> goff(pp.ops.size(), -1);
        for (const DevSweep& sw : pp.sweeps)
            for (int o = sw.op_begin; o < sw.op_end; ++o)
                if (pp.ops[o].moff >= 0) goff[o] = sw.mbase + pp.ops[o].moff;
        if ((ce = upload(pi ? p->goff_bwd : p->goff_fwd, goff, s)) != cudaSuccess) return fail(ce);
    }
    if ((ce = upload(p->slot_ptr, ptr, s)) != cudaSuccess) return fail(ce);
    if ((ce = upload(p->slot_taps, taps, s)) != cudaSuccess) return fail(ce);
    if ((ce = upload(p->slot_coef, coef, s)) != cudaSuccess) return fail(ce);
    if ((ce = cudaStreamSynchronize(s)) != cudaSuccess) return fail(ce);
    const char* jit_env = std::getenv("QF_JIT");
    if (!(jit_env && jit_env[0] == '0') && !p->plan.gates.empty()) {
        p->use_jit = jit_build(p->plan, p->jf, p->jb, p->jst);
        if (!p->use_jit && jit_env && jit_env[0] == '2') {  // QF_JIT=2: specialised kernels required
            std::string why = p->jst.error;
            delete p;
            return set_err(QF_ERUNTIME, "JIT required but unavailable: " + why);
        }
    }
    *out = p;
    return QF_OK;
}

int qf_program_jit_status(const qf_program* p, int* active, int* compiled, int* cached, double* seconds,
                          const char** error) {
    if (!p) return set_err(QF_EINVAL, "null program");
    if (active) *active = p->use_jit ? 1 : 0;
    if (compiled) *compiled = p->jst.compiled;
    if (cached) *cached = p->jst.cached;
    if (seconds) *seconds = p->jst.seconds;
    if (error) *error = p->jst.error.c_str();
    return QF_OK;
}

int qf_program_set_initial_state(qf_program* p, const double* amps) {
    if (!p || !amps) return set_err(QF_EINVAL, "qf_program_set_initial_state: null argument");
    const size_t N = size_t(1) << p->plan.n;
    cudaSetDevice(p->ctx->device);
    if (p->plan.prec == QF_C128) {
        QF_CUDA(p->init.reserve(N * 16));
        QF_CUDA(cudaMemcpy(p->init.p, amps, N * 16, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(2 * N);
        for (size_t i = 0; i < 2 * N; ++i) f[i] = (float)amps[i];
        QF_CUDA(p->init.reserve(N * 8));
        QF_CUDA(cudaMemcpy(p->init.p, f.data(), N * 8, cudaMemcpyHostToDevice));
    }
    p->has_init = true;
    return QF_OK;
}

int qf_program_destroy(qf_program* p) {
    if (!p) return QF_OK;
    cudaSetDevice(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    for (DevBuf* b : {&p->gates, &p->cmats, &p->fwd.phases, &p->fwd.ops, &p->bwd.phases, &p->bwd.ops,
                      &p->slot_ptr, &p->slot_taps, &p->slot_coef, &p->goff_fwd, &p->goff_bwd, &p->init})
        b->release();
    delete p;
    return QF_OK;
}

static int build_plan_from_ops(int n, int n_ops, const qf_op* ops, const double* mats, int n_mats, int n_params,
                               int precision, ProgramPlan& P) {
    if (n_ops < 0 || (n_ops > 0 && !ops)) return set_err(QF_EINVAL, "bad ops");
    std::vector<GateSpec> specs(n_ops);
    for (int i = 0; i < n_ops; ++i)
        specs[i] = GateSpec{ops[i].kind, ops[i].q0, ops[i].q1, ops[i].slot, ops[i].coef, ops[i].offset, ops[i].mat};
    std::string e = build_program_plan(n, specs, mats, n_mats, n_params, precision, P);
    if (!e.empty()) return set_err(QF_EINVAL, e);
    return QF_OK;
}

int qf_plan_describe(int n, int n_ops, const qf_op* ops, const double* mats, int n_mats, int n_params,
                     int precision, char* buf, size_t buflen, size_t* needed) {
    ProgramPlan P;
    int rc = build_plan_from_ops(n, n_ops, ops, mats, n_mats, n_params, precision, P);
    if (rc) return rc;
    std::string s = "{\"n\":" + std::to_string(n) + ",\"passes\":{";
    for (int pi = 0; pi < 2; ++pi) {
        const PassPlan& pp = pi ? P.bwd : P.fwd;
        s += std::string(pi ? "," : "") + (pi ? "\"bwd\"" : "\"fwd\"") + ":{\"k\":" + std::to_string(pp.k) +
             ",\"R\":" + std::to_string(pp.R) + ",\"n_taps\":" + std::to_string(pp.n_taps) + ",\"sweeps\":[";
        for (size_t si = 0; si < pp.sweeps.size(); ++si) {
            const DevSweep& sw = pp.sweeps[si];
            s += std::string(si ? "," : "") + "{\"tile_bits\":[";
            for (int t = 0; t < sw.k; ++t) s += std::string(t ? "," : "") + std::to_string(sw.tb[t]);
            s += "],\"tap_begin\":" + std::to_string(sw.tap_begin) + ",\"phases\":[";
            for (int f = 0; f < sw.n_phases; ++f) {
                const DevPhase& ph = pp.phases[sw.phase_begin + f];
                s += std::string(f ? "," : "") + "{\"reg_bits\":[";
                for (int r = 0; r < pp.R; ++r) s += std::string(r ? "," : "") + std::to_string(sw.tb[(int)ph.reg_tl[r]]);
                s += "],\"ops\":[";
                for (int o = ph.op_begin; o < ph.op_end; ++o) {
                    const DevOp& op = pp.ops[o];
                    s += std::string(o > ph.op_begin ? "," : "") + "[" + std::to_string(op.kind) + "," +
                         std::to_string(op.gate) + "," + std::to_string(op.tap) + "]";
                }
                s += "]}";
            }
            s += "]}";
        }
        s += "],\"taps\":[";
        for (size_t t = 0; t < pp.taps.size(); ++t)
            s += std::string(t ? "," : "") + "[" + std::to_string(pp.taps[t].slot) + "," + std::to_string(pp.taps[t].coef) + "]";
        s += "]}";
    }
    s += "}}";
    if (needed) *needed = s.size() + 1;
    if (buf && buflen > 0) {
        const size_t m = std::min(buflen - 1, s.size());
        std::memcpy(buf, s.data(), m);
        buf[m] = 0;
        if (m < s.size()) return set_err(QF_EINVAL, "qf_plan_describe: buffer too small");
    }
    return QF_OK;
}

int qf_jit_compile_check(int n, int n_ops, const qf_op* ops, const double* mats, int n_mats, int n_params,
                         int precision, int* kernels) {
    ProgramPlan P;
    int rc = build_plan_from_ops(n, n_ops, ops, mats, n_mats, n_params, precision, P);
    if (rc) return rc;
    int count = 0;
    for (int pi = 0; pi < 2; ++pi) {
        const PassPlan& pp = pi ? P.bwd : P.fwd;
        for (size_t si = 0; si < pp.sweeps.size(); ++si) {
            std::string cubin, err;
            if (!jit_compile_source(jit_source(P, pp, (int)si, pi == 1), cubin, err))
                return set_err(QF_ERUNTIME, err);
            ++count;
        }
    }
    if (kernels) *kernels = count;
    return QF_OK;
}

int qf_jit_hpsi_check(int n, int n_terms, const int8_t* codes, const double* w_re, const double* w_im, int precision,
                      int* compiled) {
    if (n < 1 || n > 32 || n_terms < 0 || (n_terms > 0 && (!codes || !w_re)))
        return set_err(QF_EINVAL, "qf_jit_hpsi_check: bad arguments");
    if (precision != QF_C64 && precision != QF_C128) return set_err(QF_EINVAL, "qf_jit_hpsi_check: bad precision");
    std::vector<double> wi(w_im ? std::vector<double>(w_im, w_im + n_terms) : std::vector<double>(n_terms, 0.0));
    ObservablePlan plan;
    const std::string e = build_observable_plan(n, n_terms, codes, w_re, wi.data(), geometry(precision, n).kh, plan);
    if (!e.empty()) return set_err(QF_EINVAL, e);
    if (compiled) *compiled = 0;
    if ((int)plan.terms.size() > kJitHpsiMaxTerms) return QF_OK;
    std::string cubin, err;
    if (!jit_compile_source(jit_hpsi_source(plan, precision), cubin, err)) return set_err(QF_ERUNTIME, err);
    if (compiled) *compiled = 1;
    return QF_OK;
}

int qf_program_info(const qf_program* p, int* fs, int* bs, int* fk, int* bk) {
    if (!p) return set_err(QF_EINVAL, "null program");
    if (fs) *fs = (int)p->plan.fwd.sweeps.size();
    if (bs) *bs = (int)p->plan.bwd.sweeps.size();
    if (fk) *fk = p->plan.fwd.k;
    if (bk) *bk = p->plan.bwd.k;
    return QF_OK;
}

int qf_observable_create(qf_ctx* ctx, int n, int n_terms, const int8_t* codes, const double* w_re,
                         const double* w_im, qf_observable** out) {
    if (!ctx || !out) return set_err(QF_EINVAL, "qf_observable_create: null argument");
    if (n < 1 || n > 32) return set_err(QF_EINVAL, "observable: qubit count must be in [1, 32]");
    if (n_terms < 0 || (n_terms > 0 && (!codes || !w_re)))
        return set_err(QF_EINVAL, "qf_observable_create: bad terms");
    qf_observable* o = new qf_observable();
    static std::atomic<uint64_t> next_uid{1};
    o->ctx = ctx;
    o->n = n;
    o->uid = next_uid++;
    o->codes.assign(codes, codes + (size_t)n_terms * n);
    o->w_re.assign(w_re, w_re + n_terms);
    o->w_im.assign(n_terms, 0.0);
    if (w_im) o->w_im.assign(w_im, w_im + n_terms);
    // validate now (PauliSum::add semantics, pauli.cpp:12-18)
    ObservablePlan tmp;
    std::string e = build_observable_plan(n, n_terms, o->codes.data(), o->w_re.data(), o->w_im.data(), n, tmp);
    if (!e.empty()) {
        delete o;
        return set_err(QF_EINVAL, e);
    }
    *out = o;
    return QF_OK;
}

int qf_observable_set_sharding(qf_observable* o, int mode) {
    if (!o || (mode != QF_SHARD_BATCH && mode != QF_SHARD_TERMS))
        return set_err(QF_EINVAL, "qf_observable_set_sharding: bad arguments");
    o->term_shard = mode == QF_SHARD_TERMS;
    return QF_OK;
}

int qf_observable_destroy(qf_observable* o) {
    if (!o) return QF_OK;
    cudaSetDevice(o->ctx->device);
    cudaStreamSynchronize(o->ctx->stream);
    for (auto* d : {&o->dev[0], &o->dev[1], &o->shard_dev[0], &o->shard_dev[1]}) {
        d->groups.release();
        d->terms.release();
    }
    delete o;
    return QF_OK;
}

static int stage_thetas(qf_ctx* ctx, const qf_program* prog, int batch, const double* thetas) {
    const size_t bytes = std::max<size_t>(16, (size_t)batch * prog->plan.n_params * sizeof(double));
    QF_CUDA(ctx->thetas.reserve(bytes));
    if ((size_t)batch * prog->plan.n_params > 0) {
        QF_CUDA(ctx->pin.reserve(bytes));
        std::memcpy(ctx->pin.p, thetas, (size_t)batch * prog->plan.n_params * sizeof(double));
        QF_CUDA(cudaMemcpyAsync(ctx->thetas.p, ctx->pin.p, (size_t)batch * prog->plan.n_params * sizeof(double),
                                cudaMemcpyHostToDevice, ctx->stream));
    }
    return QF_OK;
}

// Forward pass of one parameter row (device theta) into ctx->psi (state 0).
static int forward_one(qf_ctx* ctx, qf_program* prog, const double* d_theta) {
    const int n = prog->plan.n;
    const ProgramPlan& P = prog->plan;
    const size_t N = size_t(1) << n;
    const size_t vs = vsize(P.prec);
    QF_CUDA(ctx->psi.reserve(N * vs));
    cudaStream_t s = ctx->stream;
    if (prog->has_init) {
        QF_CUDA(launch_init_state(P.prec, ctx->psi.p, prog->init.p, n, 1, s));
    } else if (P.fwd.sweeps.empty()) {
        QF_CUDA(cudaMemsetAsync(ctx->psi.p, 0, N * vs, s));
        if (P.prec == QF_C128) {
            static const double one[2] = {1.0, 0.0};
            QF_CUDA(cudaMemcpyAsync(ctx->psi.p, one, 16, cudaMemcpyHostToDevice, s));
        } else {
            static const float one[2] = {1.0f, 0.0f};
            QF_CUDA(cudaMemcpyAsync(ctx->psi.p, one, 8, cudaMemcpyHostToDevice, s));
        }
    }
    SweepArgs sa{};
    sa.psi = ctx->psi.p;
    sa.theta = d_theta;
    sa.P = P.n_params;
    sa.n = n;
    sa.gates = (const DevGate*)prog->gates.p;
    sa.cmats = (const double*)prog->cmats.p;
    QF_CUDA(ctx->gmat.reserve(std::max<size_t>(16, (size_t)(P.fwd.total_mat + P.bwd.total_mat) * vs)));
    sa.gmat = ctx->gmat.p;
    sa.gmat_stride = P.fwd.total_mat + P.bwd.total_mat;
    sa.gmat_pass_base = 0;
    QF_CUDA(launch_mats(P.prec, false, (const DevOp*)prog->fwd.ops.p, (const int*)prog->goff_fwd.p,
                        (int)P.fwd.ops.size(), sa.gates, sa.cmats, sa.theta, P.n_params, 0, ctx->gmat.p,
                        sa.gmat_stride, 0, 1, s));
    sa.phases = (const DevPhase*)prog->fwd.phases.p;
    sa.ops = (const DevOp*)prog->fwd.ops.p;
    for (size_t i = 0; i < P.fwd.sweeps.size(); ++i) {
        sa.sw = P.fwd.sweeps[i];
        sa.from_zero = (i == 0 && !prog->has_init) ? 1 : 0;
        if (prog->use_jit)
            QF_CUDA((cudaError_t)jit_launch(prog->jf.sweeps[i], sa, 1 << (n - sa.sw.k), 1, s));
        else
            QF_CUDA(launch_sweep(P.prec, false, sa, 1, P.fwd.max_mat, 0, s));
        ctx->launches++;
    }
    return QF_OK;
}

static void reset_stats(qf_ctx* ctx) {
    resolve_events(ctx);
    ctx->launches = 0;
    for (int i = 0; i < 4; ++i) {
        ctx->ms[i] = ctx->bytes[i] = 0;
        ctx->class_launches[i] = 0;
    }
}

int qf_energy_grad_batch(qf_ctx* ctx, const qf_program* cprog, const qf_observable* cobs, int batch,
                         const double* thetas, double* energies, double* grads) {
    qf_program* prog = const_cast<qf_program*>(cprog);
    qf_observable* obs = const_cast<qf_observable*>(cobs);
    if (!ctx || !prog || !obs || batch < 0 || (batch > 0 && (!energies || (!thetas && prog->plan.n_params))))
        return set_err(QF_EINVAL, "qf_energy_grad_batch: bad arguments");
    if (batch == 0) return QF_OK;
    if (grads && !prog->plan.adjoint_ok) return set_err(QF_EINVAL, prog->plan.adjoint_error);
    int rc = check_thetas(prog, batch, thetas);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    const int P = prog->plan.n_params;
    rc = stage_thetas(ctx, prog, batch, thetas);
    if (rc) return rc;
    // output: [E (batch)] [G (batch x P)]
    const size_t out_n = (size_t)batch * (1 + (grads ? P : 0));
    QF_CUDA(ctx->out.reserve(out_n * 8));
    double* dE = (double*)ctx->out.p;
    double* dG = grads ? dE + batch : nullptr;
    const bool sharded = ctx->comm != nullptr;
    const bool term_shard = sharded && obs->term_shard;
    if (sharded && !term_shard) {
        // batch sharding: rank r owns rows [b0, b1); zero elsewhere; one all-reduce (exact: x + 0 = x)
        const int b0 = (int)((long long)batch * ctx->rank / ctx->world);
        const int b1 = (int)((long long)batch * (ctx->rank + 1) / ctx->world);
        QF_CUDA(cudaMemsetAsync(ctx->out.p, 0, out_n * 8, ctx->stream));
        if (b1 > b0) {
            // evaluate rows b0..b1 into temp area then scatter: reuse thetas offset via pointer arithmetic
            rc = eval_device(ctx, prog, obs, b1 - b0, (const double*)ctx->thetas.p + (size_t)b0 * P, dE + b0,
                             nullptr, dG ? dG + (size_t)b0 * P : nullptr, false);
            if (rc) return rc;
        }
    } else {
        rc = eval_device(ctx, prog, obs, batch, (const double*)ctx->thetas.p, dE, nullptr, dG, term_shard);
        if (rc) return rc;
    }
    if (sharded) {
        int r = g_nccl.allReduce(ctx->out.p, ctx->out.p, out_n, kNcclFloat64, kNcclSum, ctx->comm, ctx->stream);
        if (r) return set_err(QF_ENCCL, std::string("ncclAllReduce: ") + g_nccl.errStr(r));
    }
    QF_CUDA(ctx->pin.reserve(out_n * 8));
    QF_CUDA(cudaMemcpyAsync(ctx->pin.p, ctx->out.p, out_n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    QF_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(energies, ctx->pin.p, (size_t)batch * 8);
    if (grads) std::memcpy(grads, (double*)ctx->pin.p + batch, (size_t)batch * P * 8);
    return QF_OK;
}

int qf_energy_grad_batch_device(qf_ctx* ctx, const qf_program* cprog, const qf_observable* cobs, int batch,
                                const double* d_thetas, double* d_energies, double* d_grads) {
    qf_program* prog = const_cast<qf_program*>(cprog);
    qf_observable* obs = const_cast<qf_observable*>(cobs);
    if (!ctx || !prog || !obs || batch < 0 || (batch > 0 && !d_energies))
        return set_err(QF_EINVAL, "qf_energy_grad_batch_device: bad arguments");
    if (batch == 0) return QF_OK;
    cudaSetDevice(ctx->device);
    return eval_device(ctx, prog, obs, batch, d_thetas, d_energies, nullptr, d_grads, false);
}

int qf_run_state(qf_ctx* ctx, const qf_program* cprog, const double* theta, int guard_log2, double* amps_out) {
    qf_program* prog = const_cast<qf_program*>(cprog);
    if (!ctx || !prog || !amps_out || (!theta && prog->plan.n_params))
        return set_err(QF_EINVAL, "qf_run_state: bad arguments");
    const int n = prog->plan.n;
    if (!(std::pow(2.0, n) <= std::pow(2.0, (double)guard_log2)))  // circuit.cpp:305-307
        return set_err(QF_EINVAL, "run: state dimension exceeds memory guard");
    int rc = check_thetas(prog, 1, theta);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    rc = stage_thetas(ctx, prog, 1, theta);
    if (rc) return rc;
    rc = forward_one(ctx, prog, (const double*)ctx->thetas.p);
    if (rc) return rc;
    const ProgramPlan& P = prog->plan;
    const size_t N = size_t(1) << n;
    const size_t vs = vsize(P.prec);
    cudaStream_t s = ctx->stream;
    // Shear-form rotations (DK_RS) may apply -R: a global sign, irrelevant to
    // energies and gradients but not to the state itself -- undo it here.
    double sign = 1.0;
    {
        std::vector<unsigned char> tab((size_t)P.fwd.total_mat * vs);
        if (!tab.empty())
            QF_CUDA(cudaMemcpyAsync(tab.data(), ctx->gmat.p, tab.size(), cudaMemcpyDeviceToHost, s));
        QF_CUDA(cudaStreamSynchronize(s));
        for (const DevSweep& sw : P.fwd.sweeps)
            for (int o = sw.op_begin; o < sw.op_end; ++o) {
                const DevOp& op = P.fwd.ops[o];
                if (op.kind != DK_RS) continue;
                const size_t e = (size_t)(sw.mbase + op.moff + 1);
                const double sg = P.prec == QF_C128 ? reinterpret_cast<const double*>(tab.data())[2 * e]
                                                    : reinterpret_cast<const float*>(tab.data())[2 * e];
                if (sg < 0) sign = -sign;
            }
    }
    if (P.prec == QF_C128) {
        QF_CUDA(cudaMemcpyAsync(amps_out, ctx->psi.p, N * 16, cudaMemcpyDeviceToHost, s));
        QF_CUDA(cudaStreamSynchronize(s));
        if (sign < 0)
            for (size_t i = 0; i < 2 * N; ++i) amps_out[i] = -amps_out[i];
    } else {
        std::vector<float> f(2 * N);
        QF_CUDA(cudaMemcpyAsync(f.data(), ctx->psi.p, N * 8, cudaMemcpyDeviceToHost, s));
        QF_CUDA(cudaStreamSynchronize(s));
        for (size_t i = 0; i < 2 * N; ++i) amps_out[i] = sign * f[i];
    }
    return QF_OK;
}

int qf_sparse_energy(qf_ctx* ctx, const qf_program* cprog, int batch, const double* thetas, int64_t dim, int64_t nnz,
                     const int64_t* rows, const int64_t* cols, const double* vals, int coo_on_device,
                     double* energies) {
    // reference variational.cpp:45-52 (energy(ansatz, theta, SparseCOO)) and sparse.cpp:44-51
    qf_program* prog = const_cast<qf_program*>(cprog);
    if (!ctx || !prog || batch < 0 || nnz < 0 || (batch > 0 && (!energies || (!thetas && prog->plan.n_params))) ||
        (nnz > 0 && (!rows || !cols || !vals)))
        return set_err(QF_EINVAL, "qf_sparse_energy: bad arguments");
    const int n = prog->plan.n;
    if (dim != ((int64_t)1 << n)) return set_err(QF_EINVAL, "energy: Hamiltonian dimension mismatch");
    if (batch == 0) return QF_OK;
    int rc = check_thetas(prog, batch, thetas);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    rc = stage_thetas(ctx, prog, batch, thetas);
    if (rc) return rc;
    const int64_t *dr = rows, *dc = cols;
    const double2* dv = reinterpret_cast<const double2*>(vals);
    if (!coo_on_device && nnz > 0) {
        QF_CUDA(ctx->coo_rows.reserve((size_t)nnz * 8));
        QF_CUDA(ctx->coo_cols.reserve((size_t)nnz * 8));
        QF_CUDA(ctx->coo_vals.reserve((size_t)nnz * 16));
        QF_CUDA(cudaMemcpyAsync(ctx->coo_rows.p, rows, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
        QF_CUDA(cudaMemcpyAsync(ctx->coo_cols.p, cols, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
        QF_CUDA(cudaMemcpyAsync(ctx->coo_vals.p, vals, (size_t)nnz * 16, cudaMemcpyHostToDevice, s));
        dr = (const int64_t*)ctx->coo_rows.p;
        dc = (const int64_t*)ctx->coo_cols.p;
        dv = (const double2*)ctx->coo_vals.p;
    }
    const int blocks = coo_energy_blocks(nnz);
    QF_CUDA(ctx->epart.reserve((size_t)blocks * 8));
    QF_CUDA(ctx->out.reserve((size_t)batch * 8));
    double* d_out = (double*)ctx->out.p;
    for (int b = 0; b < batch; ++b) {
        rc = forward_one(ctx, prog, (const double*)ctx->thetas.p + (size_t)b * prog->plan.n_params);
        if (rc) return rc;
        if (nnz > 0) {
            QF_CUDA(launch_coo_energy(prog->plan.prec, dr, dc, dv, nnz, ctx->psi.p, (double*)ctx->epart.p, s));
            ReduceArgs ra{};
            ra.part = (const double*)ctx->epart.p;
            ra.count = 1;
            ra.tiles = blocks;
            ra.out = d_out + b;
            QF_CUDA(launch_reduce(ra, 1, s));
            ctx->launches += 2;
        } else {
            QF_CUDA(cudaMemsetAsync(d_out + b, 0, 8, s));
        }
    }
    QF_CUDA(cudaMemcpyAsync(energies, d_out, (size_t)batch * 8, cudaMemcpyDeviceToHost, s));
    QF_CUDA(cudaStreamSynchronize(s));
    return QF_OK;
}

int qf_expectation(qf_ctx* ctx, const qf_program* cprog, const qf_observable* cobs, const double* theta,
                   double* out_re_im) {
    qf_program* prog = const_cast<qf_program*>(cprog);
    qf_observable* obs = const_cast<qf_observable*>(cobs);
    if (!ctx || !prog || !obs || !out_re_im || (!theta && prog->plan.n_params))
        return set_err(QF_EINVAL, "qf_expectation: bad arguments");
    int rc = check_thetas(prog, 1, theta);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    rc = stage_thetas(ctx, prog, 1, theta);
    if (rc) return rc;
    QF_CUDA(ctx->out.reserve(32));
    double* dE = (double*)ctx->out.p;
    rc = eval_device(ctx, prog, obs, 1, (const double*)ctx->thetas.p, dE, dE + 1, nullptr, false);
    if (rc) return rc;
    QF_CUDA(cudaMemcpyAsync(out_re_im, dE, 16, cudaMemcpyDeviceToHost, ctx->stream));
    QF_CUDA(cudaStreamSynchronize(ctx->stream));
    return QF_OK;
}

int qf_adam_step_device(qf_ctx* ctx, int batch, int P, double* th, double* m, double* v, const double* g,
                        int t, double lr, double b1, double b2, double eps) {
    if (!ctx || batch < 0 || P < 0 || t < 1) return set_err(QF_EINVAL, "qf_adam_step_device: bad arguments");
    cudaSetDevice(ctx->device);
    const double c1 = 1.0 - std::pow(b1, t);
    const double c2 = 1.0 - std::pow(b2, t);
    QF_CUDA(launch_adam(batch * P, th, m, v, g, lr, b1, b2, eps, c1, c2, ctx->stream));
    return QF_OK;
}

int qf_pauli_sum_to_coo(qf_ctx* ctx, const qf_observable* obs, int n_guard, int device_buffers, int64_t* rows,
                        int64_t* cols, double* vals, int64_t capacity, int64_t* nnz) {
    // reference src/pauli.cpp:89-153
    if (!ctx || !obs || !nnz) return set_err(QF_EINVAL, "qf_pauli_sum_to_coo: null argument");
    const int n = obs->n;
    if (n < 1) return set_err(QF_EINVAL, "pauli_sum_to_coo: empty system");
    if (n > n_guard) return set_err(QF_EINVAL, "pauli_sum_to_coo: qubit count exceeds memory guard");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const int T = (int)obs->w_re.size();
    if (T == 0) {
        *nnz = 0;
        return QF_OK;
    }
    const int64_t dim = (int64_t)1 << n;
    int64_t* offsets = nullptr;
    int64_t total = 0;
    if (ctx->coo_uid == obs->uid) {  // sizing call already counted this observable: reuse its offsets
        offsets = (int64_t*)ctx->coo_off.p + dim + 1;
        total = ctx->coo_total;
    } else {
    ctx->coo_uid = 0;
    // group terms by flip mask (ascending), input order inside a group
    std::map<uint64_t, std::vector<CooTerm>> by_flip;
    static const double ip[4][2] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    for (int t = 0; t < T; ++t) {
        uint64_t flip = 0, z = 0;
        int y = 0;
        for (int i = 0; i < n; ++i) {
            const int c = obs->codes[(size_t)t * n + i];
            const uint64_t bit = 1ull << (n - 1 - i);
            if (c == 1) flip |= bit;
            if (c == 2) { flip |= bit; z |= bit; ++y; }
            if (c == 3) z |= bit;
        }
        const double wr = obs->w_re[t], wi = obs->w_im[t];
        CooTerm ct;
        ct.z = z;
        ct.c_re = wr * ip[y & 3][0] - wi * ip[y & 3][1];
        ct.c_im = wr * ip[y & 3][1] + wi * ip[y & 3][0];
        by_flip[flip].push_back(ct);
    }
    std::vector<CooGroup> groups;
    std::vector<CooTerm> terms;
    for (auto& [f, ts] : by_flip) {
        CooGroup g;
        g.flip = f;
        g.term_begin = (int)terms.size();
        terms.insert(terms.end(), ts.begin(), ts.end());
        g.term_end = (int)terms.size();
        groups.push_back(g);
    }
    // flip-trie rank events for the tiled writer (groups ascend by flip; kernels.cuh CooEvent)
    std::vector<CooEvent> events;
    if (groups.size() <= 32) {
        auto bits = [](int a, int b) { return (uint32_t)((((uint64_t)1 << b) - 1) & ~(((uint64_t)1 << a) - 1)); };
        std::vector<std::array<int, 2>> stack{{0, (int)groups.size()}};
        while (!stack.empty()) {
            const auto [lo, hi] = stack.back();
            stack.pop_back();
            if (hi - lo < 2) continue;
            const int d = 63 - __builtin_clzll(groups[lo].flip ^ groups[hi - 1].flip);
            int mid = lo;
            while (!((groups[mid].flip >> d) & 1)) ++mid;
            events.push_back({lo, d, 1, bits(mid, hi)});
            events.push_back({mid, d, -1, bits(lo, hi)});
            events.push_back({hi, d, 1, bits(lo, mid)});
            stack.push_back({lo, mid});
            stack.push_back({mid, hi});
        }
        std::stable_sort(events.begin(), events.end(),
                         [](const CooEvent& x, const CooEvent& y) { return x.pos < y.pos; });
    }
    if (events.empty()) events.push_back({1 << 30, 0, 0, 0});
    ctx->coo_n_events = (int)events.size();
    QF_CUDA(upload(ctx->coo_nodes, events, s));
    QF_CUDA(upload(ctx->coo_groups, groups, s));
    QF_CUDA(upload(ctx->coo_terms, terms, s));
    QF_CUDA(ctx->coo_off.reserve((size_t)(2 * dim + 2) * 8));  // counts [dim + 1] then offsets [dim + 1]
    int64_t* counts = (int64_t*)ctx->coo_off.p;
    offsets = counts + dim + 1;
    QF_CUDA(cudaMemsetAsync(counts + dim, 0, 8, s));
    QF_CUDA(launch_coo_count((const CooGroup*)ctx->coo_groups.p, (int)groups.size(),
                             (const CooTerm*)ctx->coo_terms.p, (int)terms.size(), n, counts, s));
    size_t scratch = 0;
    QF_CUDA(coo_scan(counts, offsets, dim, nullptr, &scratch, s));
    QF_CUDA(ctx->coo_scratch.reserve(std::max<size_t>(scratch, 16)));
    QF_CUDA(coo_scan(counts, offsets, dim, ctx->coo_scratch.p, &scratch, s));
    QF_CUDA(cudaMemcpyAsync(&total, offsets + dim, 8, cudaMemcpyDeviceToHost, s));
    QF_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 2;
    ctx->coo_uid = obs->uid;
    ctx->coo_n_groups = (int)groups.size();
    ctx->coo_n_terms = (int)terms.size();
    ctx->coo_total = total;
    }
    *nnz = total;
    if (!rows && !cols && !vals) return QF_OK;
    if (!rows || !cols || !vals || capacity < total)
        return set_err(QF_EINVAL, "qf_pauli_sum_to_coo: output buffers missing or too small");
    int64_t *dr = rows, *dc = cols;
    double2* dv = reinterpret_cast<double2*>(vals);
    if (!device_buffers) {
        QF_CUDA(ctx->coo_rows.reserve(std::max<size_t>(16, (size_t)total * 8)));
        QF_CUDA(ctx->coo_cols.reserve(std::max<size_t>(16, (size_t)total * 8)));
        QF_CUDA(ctx->coo_vals.reserve(std::max<size_t>(16, (size_t)total * 16)));
        dr = (int64_t*)ctx->coo_rows.p;
        dc = (int64_t*)ctx->coo_cols.p;
        dv = (double2*)ctx->coo_vals.p;
    }
    QF_CUDA(launch_coo_write((const CooGroup*)ctx->coo_groups.p, ctx->coo_n_groups, (const CooTerm*)ctx->coo_terms.p,
                             ctx->coo_n_terms, (const CooEvent*)ctx->coo_nodes.p, ctx->coo_n_events, n, offsets, dr, dc, dv, s));
    ctx->launches += 1;
    if (!device_buffers && total > 0) {
        QF_CUDA(cudaMemcpyAsync(rows, dr, (size_t)total * 8, cudaMemcpyDeviceToHost, s));
        QF_CUDA(cudaMemcpyAsync(cols, dc, (size_t)total * 8, cudaMemcpyDeviceToHost, s));
        QF_CUDA(cudaMemcpyAsync(vals, dv, (size_t)total * 16, cudaMemcpyDeviceToHost, s));
    }
    QF_CUDA(cudaStreamSynchronize(s));
    return QF_OK;
}

int qf_mipt_haar(qf_ctx* ctx, int n, int depth, double p, int trajectories, uint64_t seed, int precision,
                 double* entropies, long long* n_measurements) {
    // reference experiments.cpp:210-250 (exp_mipt_haar) with circuit.cpp:391-429 (measure_collapse),
    // :431-470 (subsystem_entropy of qubits [0, n/2)) and :472-489 (haar_su4)
    if (!ctx || !entropies) return set_err(QF_EINVAL, "qf_mipt_haar: null argument");
    if (n < 2 || n > 20) return set_err(QF_EINVAL, "mipt-haar: N must lie in [2, 20]");
    if (!(p >= 0.0 && p <= 1.0)) return set_err(QF_EINVAL, "mipt-haar: p must lie in [0, 1]");
    if (trajectories < 1) return set_err(QF_EINVAL, "mipt-haar: trajectories must be >= 1");
    if (precision != QF_C64 && precision != QF_C128) return set_err(QF_EINVAL, "qf_mipt_haar: bad precision");
    depth = std::max(depth, 0);
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const bool tm = std::getenv("QF_MIPT_TIMING") != nullptr;  // development: phase timings on stderr
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    double t_gen = 0, t_circ = 0, t_ent = 0;
    auto T0 = now();
    const int npmax = n / 2;
    const size_t mat_doubles = (size_t)npmax * 32;  // per state and layer

    // ---- host randomness, in the reference's draw order (per trajectory stream)
    struct Meas {
        int layer, pos;
        double u;
    };
    std::vector<double> mats((size_t)std::max(depth, 1) * trajectories * mat_doubles, 0.0);
    std::vector<std::vector<Meas>> meas(trajectories);
    {
        const auto streams = qforge::RngStream(seed).split((size_t)trajectories);
        auto work = [&](int t0, int t1) {
            for (int tr = t0; tr < t1; ++tr) {
                qforge::RngStream rs = streams[tr];
                for (int layer = 0; layer < depth; ++layer) {
                    int j = 0;
                    for (int i = layer % 2; i + 1 < n; i += 2, ++j) {
                        cd q[4][4];
                        haar_su4(rs, q);
                        double* m = mats.data() + ((size_t)layer * trajectories + tr) * mat_doubles + (size_t)j * 32;
                        for (int r = 0; r < 4; ++r)
                            for (int c = 0; c < 4; ++c) {
                                m[(r * 4 + c) * 2] = q[r][c].real();
                                m[(r * 4 + c) * 2 + 1] = q[r][c].imag();
                            }
                    }
                    for (int qb = 0; qb < n; ++qb)
                        if (rs.uniform() < p) meas[tr].push_back({layer, n - 1 - qb, rs.uniform()});
                }
            }
        };
        const int nthr = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), trajectories));
        std::vector<std::thread> pool;
        for (int t = 0; t < nthr; ++t)
            pool.emplace_back(work, (int)((long long)trajectories * t / nthr),
                              (int)((long long)trajectories * (t + 1) / nthr));
        for (auto& th : pool) th.join();
    }
    long long total_meas = 0;
    for (auto& v : meas) total_meas += (long long)v.size();
    t_gen = secs(T0, now());
    if (n_measurements) *n_measurements = total_meas;

    // ---- layer programs: brickwork of dense two-qubit gates, matrices per state
    qf_program* progs[2] = {nullptr, nullptr};
    struct ProgGuard {
        qf_program** p;
        ~ProgGuard() {
            for (int i = 0; i < 2; ++i)
                if (p[i]) qf_program_destroy(p[i]);
        }
    } guard{progs};
    std::vector<double> dummy;
    for (int k = 0; k < 4; ++k)  // a dense unitary (classified as a general gate; replaced per state)
        for (int l = 0; l < 4; ++l) {
            const double ang = 2.0 * M_PI * k * l / 4.0;
            dummy.push_back(0.5 * std::cos(ang));
            dummy.push_back(0.5 * std::sin(ang));
        }
    for (int par = 0; par < 2; ++par) {
        std::vector<qf_op> ops;
        std::vector<double> ms;
        int j = 0;
        for (int i = par; i + 1 < n; i += 2, ++j) {
            qf_op o{};
            o.kind = QF_UNITARY;
            o.q0 = i;
            o.q1 = i + 1;
            o.slot = -1;
            o.coef = 1.0;
            o.mat = j;
            ops.push_back(o);
            ms.insert(ms.end(), dummy.begin(), dummy.end());
        }
        if (ops.empty()) continue;
        int rc = qf_program_create(ctx, n, (int)ops.size(), ops.data(), ms.data(), j, 0, precision, &progs[par]);
        if (rc) return rc;
    }

    // ---- chunks of trajectories
    const size_t N = size_t(1) << n;
    const size_t vs = vsize(precision);
    const int keep = n / 2;
    const int64_t dk = (int64_t)1 << keep, de = (int64_t)1 << (n - keep);
    size_t fr = 0, tot = 0;
    QF_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t budget = (size_t)(0.5 * (double)(fr + ctx->psi.cap));
    const size_t per_state = N * vs + (size_t)depth * mat_doubles * 8 + (1u << kMeasMax) * 8 + 256;
    int bc = (int)std::max<size_t>(1, std::min<size_t>(budget / per_state, (size_t)trajectories));
    bc = std::min(bc, 65535);
    QF_CUDA(ctx->psi.reserve((size_t)bc * N * vs));
    LocalBuf d_mats, d_rounds, d_hist, d_mask, d_bits, d_scale, d_out, d_w;
    QF_CUDA(d_mats.reserve(std::max<size_t>(16, (size_t)depth * bc * mat_doubles * 8)));
    QF_CUDA(d_rounds.reserve((size_t)bc * sizeof(MeasRound)));
    QF_CUDA(d_hist.reserve((size_t)bc * (1u << kMeasMax) * 8));
    QF_CUDA(d_mask.reserve((size_t)bc * 4));
    QF_CUDA(d_bits.reserve((size_t)bc * 4));
    QF_CUDA(d_scale.reserve((size_t)bc * 8));
    QF_CUDA(d_out.reserve((size_t)bc * kMeasMax * 4));
    QF_CUDA(d_w.reserve((size_t)bc * dk * 8));
    std::lock_guard<std::mutex> linalg_lock(g_linalg_mu);  // the eigen lanes are process-wide
    if (!g_linalg.load()) return set_err(QF_ERUNTIME, g_linalg.err);
    LinAlg& la = g_linalg;
    const int lanes = std::max(1, std::min(kEigLanes, bc));
    for (int l = 0; l < lanes; ++l) {
        int rc = lane_setup(g_lanes[l], la, ctx->device, dk, N);
        if (rc) return rc;
    }
    std::vector<double> w_host((size_t)bc * dk);
    std::vector<MeasRound> rounds(bc);
    for (int t0 = 0; t0 < trajectories; t0 += bc) {
        const int nb = std::min(bc, trajectories - t0);
        // matrices of this chunk, layer-major [depth][nb][npmax][32]
        for (int layer = 0; layer < depth; ++layer)
            QF_CUDA(cudaMemcpyAsync((double*)d_mats.p + (size_t)layer * nb * mat_doubles,
                                    mats.data() + ((size_t)layer * trajectories + t0) * mat_doubles,
                                    (size_t)nb * mat_doubles * 8, cudaMemcpyHostToDevice, s));
        QF_CUDA(launch_set_basis0(precision, ctx->psi.p, n, nb, s));
        std::vector<size_t> cursor(nb, 0);
        for (int layer = 0; layer < depth; ++layer) {
            qf_program* prog = progs[layer % 2];
            if (prog) {
                const ProgramPlan& P = prog->plan;
                SweepArgs sa{};
                sa.psi = ctx->psi.p;
                sa.n = n;
                sa.gates = (const DevGate*)prog->gates.p;
                sa.cmats = (const double*)d_mats.p + (size_t)layer * nb * mat_doubles;
                QF_CUDA(ctx->gmat.reserve(std::max<size_t>(16, (size_t)nb * P.fwd.total_mat * vs)));
                sa.gmat = ctx->gmat.p;
                sa.gmat_stride = P.fwd.total_mat;
                QF_CUDA(launch_mats(precision, false, (const DevOp*)prog->fwd.ops.p, (const int*)prog->goff_fwd.p,
                                    (int)P.fwd.ops.size(), sa.gates, sa.cmats, nullptr, 0, 0, ctx->gmat.p,
                                    sa.gmat_stride, 0, nb, s, mat_doubles));
                sa.phases = (const DevPhase*)prog->fwd.phases.p;
                sa.ops = (const DevOp*)prog->fwd.ops.p;
                for (size_t i = 0; i < P.fwd.sweeps.size(); ++i) {
                    sa.sw = P.fwd.sweeps[i];
                    if (prog->use_jit)
                        QF_CUDA((cudaError_t)jit_launch(prog->jf.sweeps[i], sa, 1 << (n - sa.sw.k), nb, s));
                    else
                        QF_CUDA(launch_sweep(precision, false, sa, nb, P.fwd.max_mat, 0, s));
                    ctx->launches++;
                }
            }
            // measurements of this layer, in rounds of up to kMeasMax per trajectory
            for (;;) {
                int maxc = 0;
                for (int b = 0; b < nb; ++b) {
                    const auto& v = meas[t0 + b];
                    MeasRound& r = rounds[b];
                    r.count = 0;
                    while (cursor[b] < v.size() && v[cursor[b]].layer == layer && r.count < kMeasMax) {
                        r.pos[r.count] = v[cursor[b]].pos;
                        r.u[r.count] = v[cursor[b]].u;
                        ++r.count;
                        ++cursor[b];
                    }
                    maxc = std::max(maxc, r.count);
                }
                if (maxc == 0) break;
                QF_CUDA(cudaMemcpyAsync(d_rounds.p, rounds.data(), (size_t)nb * sizeof(MeasRound),
                                        cudaMemcpyHostToDevice, s));
                QF_CUDA(launch_meas_hist(precision, ctx->psi.p, n, nb, (const MeasRound*)d_rounds.p, maxc,
                                         (double*)d_hist.p, s));
                QF_CUDA(launch_meas_decide((const MeasRound*)d_rounds.p, (const double*)d_hist.p, nb,
                                           (uint32_t*)d_mask.p, (uint32_t*)d_bits.p, (double*)d_scale.p,
                                           (int*)d_out.p, s));
                QF_CUDA(launch_meas_project(precision, ctx->psi.p, n, nb, (const MeasRound*)d_rounds.p,
                                            (const uint32_t*)d_mask.p, (const uint32_t*)d_bits.p,
                                            (const double*)d_scale.p, s));
                QF_CUDA(cudaStreamSynchronize(s));  // rounds[] is reused by the next upload
                ctx->launches += 3;
            }
        }
        if (tm) {
            QF_CUDA(cudaStreamSynchronize(s));
            t_circ += secs(T0, now());
            T0 = now();
        }
        // half-chain entropy: eigenvalues of A^H A, A = psi as a (de x dk) column-major
        // matrix (same spectrum as the reference's SVD of psi reshaped to dk x de)
        QF_CUDA(cudaStreamSynchronize(s));
        {
            std::vector<std::thread> pool;
            std::vector<int> lane_rc(lanes, QF_OK);
            std::vector<std::string> lane_err(lanes);
            for (int l = 0; l < lanes; ++l)
                pool.emplace_back([&, l] {
                    EigLane& L = g_lanes[l];
                    cudaSetDevice(ctx->device);
                    const double one = 1.0, zero = 0.0;
                    // double-precision spectrum for both state precisions: a complex64 CHEEVD
                    // loses the small Schmidt values (n = 20: -0.22 bits of mean entropy)
                    for (int b = l; b < nb; b += lanes) {
                        cudaError_t e = launch_convert_state(
                            precision, (const unsigned char*)ctx->psi.p + (size_t)b * N * vs, (double*)L.conv.p,
                            (int64_t)N, L.st);
                        if (e != cudaSuccess) {
                            lane_rc[l] = QF_ECUDA;
                            lane_err[l] = cudaGetErrorString(e);
                            return;
                        }
                        if (la.zherk(L.cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, (int)dk, (int)de, &one,
                                     (const cuDoubleComplex*)L.conv.p, (int)de, &zero, (cuDoubleComplex*)L.rho.p,
                                     (int)dk) != CUBLAS_STATUS_SUCCESS ||
                            la.zheevd(L.cs, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, (int)dk,
                                      (cuDoubleComplex*)L.rho.p, (int)dk, (double*)d_w.p + (size_t)b * dk,
                                      (cuDoubleComplex*)L.work.p, L.lwork, (int*)L.info.p) !=
                                CUSOLVER_STATUS_SUCCESS) {
                            lane_rc[l] = QF_ERUNTIME;
                            lane_err[l] = "cuBLAS ZHERK / cuSOLVER ZHEEVD failed";
                            return;
                        }
                    }
                    cudaError_t e = cudaStreamSynchronize(L.st);
                    if (e != cudaSuccess) {
                        lane_rc[l] = QF_ECUDA;
                        lane_err[l] = cudaGetErrorString(e);
                    }
                });
            for (auto& th : pool) th.join();
            for (int l = 0; l < lanes; ++l)
                if (lane_rc[l]) return set_err(lane_rc[l], "qf_mipt_haar: " + lane_err[l]);
        }
        QF_CUDA(cudaMemcpyAsync(w_host.data(), d_w.p, (size_t)nb * dk * 8, cudaMemcpyDeviceToHost, s));
        QF_CUDA(cudaStreamSynchronize(s));
        for (int b = 0; b < nb; ++b) {
            double ent = 0.0;
            for (int64_t i = dk - 1; i >= 0; --i) {  // descending, as the reference's singular values
                const double pr = std::clamp(w_host[(size_t)b * dk + i], 0.0, 1.0);
                if (pr > 1e-15) ent -= pr * std::log2(pr);
            }
            entropies[t0 + b] = std::max(ent, 0.0);
        }
        if (tm) {
            t_ent += secs(T0, now());
            T0 = now();
        }
    }
    if (tm) fprintf(stderr, "qf_mipt_haar: host randomness %.3f s, circuits %.3f s, entropy %.3f s\n", t_gen, t_circ, t_ent);
    return QF_OK;
}

int qf_shadow_snapshots(qf_ctx* ctx, const qf_program* cprep, const double* theta, int m, const int8_t* bases,
                        const double* u, int8_t* outcomes) {
    // reference shadows.cpp:50-85 (shadow_snapshots): per snapshot r, the prepared state
    // rotated into bases[r] (basis_rotation :33-44; 1 = X, 2 = Y, 3 = Z) and one sample
    // by inverse CDF with the uniform u[r] (= rng.split(m)[r].uniform() in the reference)
    qf_program* prep = const_cast<qf_program*>(cprep);
    if (!ctx || !prep || m < 0 || (m > 0 && (!bases || !u || !outcomes)) || (!theta && prep->plan.n_params))
        return set_err(QF_EINVAL, "qf_shadow_snapshots: bad arguments");
    const int n = prep->plan.n, prec = prep->plan.prec;
    for (size_t i = 0; i < (size_t)m * n; ++i)
        if (bases[i] < 1 || bases[i] > 3) return set_err(QF_EINVAL, "shadow_snapshots: bad basis code");
    if (m == 0) return QF_OK;
    int rc = check_thetas(prep, 1, theta);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    rc = stage_thetas(ctx, prep, 1, theta);
    if (rc) return rc;
    rc = forward_one(ctx, prep, (const double*)ctx->thetas.p);  // psi -> ctx->psi (global sign irrelevant)
    if (rc) return rc;
    // per-qubit basis program (dense single-qubit gates, matrices per snapshot)
    qf_program*& bp = ctx->basis_progs[{n, prec}];
    if (!bp) {
        std::vector<qf_op> ops(n);
        std::vector<double> ms;
        const double h = std::sqrt(0.5);
        for (int q = 0; q < n; ++q) {
            ops[q] = qf_op{};
            ops[q].kind = QF_UNITARY;
            ops[q].q0 = q;
            ops[q].q1 = -1;
            ops[q].slot = -1;
            ops[q].coef = 1.0;
            ops[q].mat = q;
            const double hx[8] = {h, 0, h, 0, h, 0, -h, 0};  // placeholder; replaced per snapshot
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) {
                    ms.push_back(r < 2 && c < 2 ? hx[(r * 2 + c) * 2] : 0.0);
                    ms.push_back(r < 2 && c < 2 ? hx[(r * 2 + c) * 2 + 1] : 0.0);
                }
        }
        rc = qf_program_create(ctx, n, n, ops.data(), ms.data(), n, 0, prec, &bp);
        if (rc) {
            bp = nullptr;
            return rc;
        }
    }
    const ProgramPlan& P = bp->plan;
    const size_t N = size_t(1) << n, vs = vsize(prec);
    size_t fr = 0, tot = 0;
    QF_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t budget = (size_t)(0.5 * (double)(fr + ctx->lam.cap));
    const int cb = sample_chunk_bits(n);
    const size_t nc = N >> cb;
    const size_t per_state = N * vs + (size_t)n * 32 * 8 + nc * 8 + 64;
    int bc = (int)std::max<size_t>(1, std::min<size_t>(budget / per_state, (size_t)m));
    bc = std::min(bc, 65535);
    QF_CUDA(ctx->lam.reserve((size_t)bc * N * vs));
    QF_CUDA(ctx->gmat.reserve(std::max<size_t>(16, (size_t)bc * P.fwd.total_mat * vs)));
    LocalBuf d_cm, d_u, d_csum, d_hit;
    QF_CUDA(d_cm.reserve((size_t)bc * n * 32 * 8));
    QF_CUDA(d_u.reserve((size_t)bc * 8));
    QF_CUDA(d_csum.reserve((size_t)bc * nc * 8));
    QF_CUDA(d_hit.reserve((size_t)bc * 8));
    const double h = std::sqrt(0.5);
    // basis_rotation: X -> [[s, s], [s, -s]], Y -> [[s, -i s], [s, i s]], Z -> identity
    const double rot[4][8] = {{0}, {h, 0, h, 0, h, 0, -h, 0}, {h, 0, 0, -h, h, 0, 0, h}, {1, 0, 0, 0, 0, 0, 1, 0}};
    std::vector<double> cm((size_t)bc * n * 32);
    std::vector<int64_t> hits(bc);
    for (int r0 = 0; r0 < m; r0 += bc) {
        const int nb = std::min(bc, m - r0);
        std::fill(cm.begin(), cm.end(), 0.0);
        for (int b = 0; b < nb; ++b)
            for (int q = 0; q < n; ++q) {
                const double* R = rot[bases[(size_t)(r0 + b) * n + q]];
                double* dst = cm.data() + ((size_t)b * n + q) * 32;
                for (int rr = 0; rr < 2; ++rr)
                    for (int c = 0; c < 2; ++c) {
                        dst[(rr * 4 + c) * 2] = R[(rr * 2 + c) * 2];
                        dst[(rr * 4 + c) * 2 + 1] = R[(rr * 2 + c) * 2 + 1];
                    }
            }
        QF_CUDA(cudaMemcpyAsync(d_cm.p, cm.data(), (size_t)nb * n * 32 * 8, cudaMemcpyHostToDevice, s));
        QF_CUDA(cudaMemcpyAsync(d_u.p, u + r0, (size_t)nb * 8, cudaMemcpyHostToDevice, s));
        QF_CUDA(launch_init_state(prec, ctx->lam.p, ctx->psi.p, n, nb, s));  // nb copies of psi
        SweepArgs sa{};
        sa.psi = ctx->lam.p;
        sa.n = n;
        sa.gates = (const DevGate*)bp->gates.p;
        sa.cmats = (const double*)d_cm.p;
        sa.gmat = ctx->gmat.p;
        sa.gmat_stride = P.fwd.total_mat;
        QF_CUDA(launch_mats(prec, false, (const DevOp*)bp->fwd.ops.p, (const int*)bp->goff_fwd.p, (int)P.fwd.ops.size(),
                            sa.gates, sa.cmats, nullptr, 0, 0, ctx->gmat.p, sa.gmat_stride, 0, nb, s,
                            (size_t)n * 32));
        sa.phases = (const DevPhase*)bp->fwd.phases.p;
        sa.ops = (const DevOp*)bp->fwd.ops.p;
        for (size_t i = 0; i < P.fwd.sweeps.size(); ++i) {
            sa.sw = P.fwd.sweeps[i];
            if (bp->use_jit)
                QF_CUDA((cudaError_t)jit_launch(bp->jf.sweeps[i], sa, 1 << (n - sa.sw.k), nb, s));
            else
                QF_CUDA(launch_sweep(prec, false, sa, nb, P.fwd.max_mat, 0, s));
            ctx->launches++;
        }
        QF_CUDA(launch_sample(prec, ctx->lam.p, n, nb, (const double*)d_u.p, (double*)d_csum.p, (int64_t*)d_hit.p, s));
        QF_CUDA(cudaMemcpyAsync(hits.data(), d_hit.p, (size_t)nb * 8, cudaMemcpyDeviceToHost, s));
        QF_CUDA(cudaStreamSynchronize(s));
        for (int b = 0; b < nb; ++b)
            for (int q = 0; q < n; ++q)
                outcomes[(size_t)(r0 + b) * n + q] = (int8_t)((hits[b] >> (n - 1 - q)) & 1);
    }
    return QF_OK;
}

int qf_noise_trajectories(qf_ctx* ctx, int n, int n_ops, const qf_op* ops, const double* mats, int n_mats,
                          const int* op_chan_ptr, const int* op_chan, const int* chan_kraus_ptr, const double* kraus,
                          const double* init, int trajectories, const double* u, int precision, double* states,
                          double* log_probs, qf_observable* obs, double* expvals) {
    // reference noise.cpp:162-197 (mc_trajectory), batched: trajectory t uses the uniforms
    // u[t][0 .. n_apps) in channel-application order (the reference draws one per application)
    if (!ctx || n < 1 || n > 30 || n_ops < 0 || (n_ops > 0 && (!ops || !op_chan_ptr)) || trajectories < 0 ||
        (precision != QF_C64 && precision != QF_C128) || (obs && !expvals) || (obs && obs->n != n))
        return set_err(QF_EINVAL, "qf_noise_trajectories: bad arguments");
    const int n_apps = n_ops ? op_chan_ptr[n_ops] : 0;
    if (n_apps > 0 && (!op_chan || !chan_kraus_ptr || !kraus || (trajectories > 0 && !u)))
        return set_err(QF_EINVAL, "qf_noise_trajectories: missing channel data");
    if (trajectories == 0) return QF_OK;
    std::vector<int> Dg(n_ops), P0(n_ops), P1(n_ops);
    std::vector<double2> gm((size_t)std::max(n_ops, 1) * 16);
    for (int j = 0; j < n_ops; ++j) {
        const qf_op& o = ops[j];
        const bool two = o.kind == QF_RZZ || o.kind == QF_CX || o.kind == QF_CZ || o.kind == QF_SU4 ||
                         (o.kind == QF_UNITARY && o.q1 >= 0);
        if (o.slot >= 0) return set_err(QF_EINVAL, "qf_noise_trajectories: constant circuits only (slot = -1)");
        if (o.q0 < 0 || o.q0 >= n || (two && (o.q1 < 0 || o.q1 >= n || o.q1 == o.q0)))
            return set_err(QF_EINVAL, "Circuit: wire out of range");
        cd m[16];
        int rc = host_gate_matrix(o, mats, n_mats, Dg[j], m);
        if (rc) return rc;
        P0[j] = n - 1 - o.q0;
        P1[j] = Dg[j] == 4 ? n - 1 - o.q1 : -1;
        for (int i = 0; i < 16; ++i) gm[(size_t)j * 16 + i] = make_double2(m[i].real(), m[i].imag());
    }
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const size_t N = size_t(1) << n, vs = vsize(precision);
    size_t fr = 0, tot = 0;
    QF_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t budget = (size_t)(0.5 * (double)(fr + ctx->lam.cap));
    int bc = (int)std::max<size_t>(1, std::min<size_t>(budget / (N * vs + 1024), (size_t)trajectories));
    bc = std::min(bc, 65535);
    QF_CUDA(ctx->lam.reserve((size_t)bc * N * vs));
    LocalBuf d_gm, d_rho, d_k, d_init, d_part, d_E;
    QF_CUDA(d_gm.reserve(gm.size() * 16));
    QF_CUDA(cudaMemcpyAsync(d_gm.p, gm.data(), gm.size() * 16, cudaMemcpyHostToDevice, s));
    const int parts = local_rho_parts(n);
    QF_CUDA(d_rho.reserve((size_t)bc * parts * 16 * 16));
    QF_CUDA(d_k.reserve((size_t)bc * 16 * 16));
    if (init) {
        QF_CUDA(d_init.reserve(N * vs));
        if (precision == QF_C128) {
            QF_CUDA(cudaMemcpyAsync(d_init.p, init, N * 16, cudaMemcpyHostToDevice, s));
        } else {
            std::vector<float> f(2 * N);
            for (size_t i = 0; i < 2 * N; ++i) f[i] = (float)init[i];
            QF_CUDA(cudaMemcpyAsync(d_init.p, f.data(), N * 8, cudaMemcpyHostToDevice, s));
            QF_CUDA(cudaStreamSynchronize(s));
        }
    }
    ObsDev* od = nullptr;
    int tiles_h = 0;
    if (obs) {
        const Geometry geo = geometry(precision, n);
        od = &obs->dev[precision];
        int rc = ensure_obs_dev(obs, precision, geo.kh, *od, 0, (int)obs->w_re.size());
        if (rc) return rc;
        tiles_h = 1 << (n - geo.kh);
        QF_CUDA(d_part.reserve((size_t)bc * tiles_h * 8));
        QF_CUDA(d_E.reserve((size_t)bc * 8));
    }
    std::vector<double2> rho((size_t)bc * parts * 16), km((size_t)bc * 16);
    std::vector<double> logp(bc);
    std::vector<float> fbuf;
    for (int t0 = 0; t0 < trajectories; t0 += bc) {
        const int nb = std::min(bc, trajectories - t0);
        if (init)
            QF_CUDA(launch_init_state(precision, ctx->lam.p, d_init.p, n, nb, s));
        else
            QF_CUDA(launch_set_basis0(precision, ctx->lam.p, n, nb, s));
        std::fill(logp.begin(), logp.end(), 0.0);
        int app = 0;
        for (int j = 0; j < n_ops; ++j) {
            const int D = Dg[j];
            QF_CUDA(launch_apply_local(precision, ctx->lam.p, n, nb, P0[j], P1[j], (const double2*)d_gm.p + (size_t)j * 16,
                                       false, s));
            ctx->launches++;
            for (int ci = op_chan_ptr[j]; ci < op_chan_ptr[j + 1]; ++ci, ++app) {
                const int ch = op_chan[ci];
                const int k0 = chan_kraus_ptr[ch], k1 = chan_kraus_ptr[ch + 1];
                if (k1 <= k0) return set_err(QF_EINVAL, "KrausChannel: no operators");
                QF_CUDA(launch_local_rho(precision, ctx->lam.p, n, nb, P0[j], P1[j], (double2*)d_rho.p, s));
                QF_CUDA(cudaMemcpyAsync(rho.data(), d_rho.p, (size_t)nb * parts * D * D * 16, cudaMemcpyDeviceToHost,
                                        s));
                QF_CUDA(cudaStreamSynchronize(s));
                for (int b = 0; b < nb; ++b) {
                    double2 r[16];
                    for (int e = 0; e < D * D; ++e) {  // parts summed in order
                        double x = 0.0, y = 0.0;
                        for (int pt = 0; pt < parts; ++pt) {
                            x += rho[((size_t)b * parts + pt) * D * D + e].x;
                            y += rho[((size_t)b * parts + pt) * D * D + e].y;
                        }
                        r[e] = make_double2(x, y);
                    }
                    std::vector<double> probs;
                    double acc = 0.0;
                    for (int k = k0; k < k1; ++k) {  // p_k = || K_k psi ||^2 = tr(K rho K^dagger)
                        const double* K = kraus + 32 * (size_t)k;
                        double pk = 0.0;
                        for (int a = 0; a < D; ++a) {
                            cd kr[4];
                            for (int i = 0; i < D; ++i) kr[i] = cd(K[(a * 4 + i) * 2], K[(a * 4 + i) * 2 + 1]);
                            cd sa = 0.0;
                            for (int i = 0; i < D; ++i)
                                for (int jj = 0; jj < D; ++jj)
                                    sa += kr[i] * cd(r[i * D + jj].x, r[i * D + jj].y) * std::conj(kr[jj]);
                            pk += sa.real();
                        }
                        probs.push_back(pk);
                        acc += pk;
                    }
                    if (!(acc > 1e-14)) return set_err(QF_EINVAL, "mc_trajectory: all branch probabilities vanish");
                    const double uu = u[(size_t)(t0 + b) * n_apps + app] * acc;
                    size_t pick = probs.size() - 1;
                    double run = 0.0;
                    for (size_t i = 0; i < probs.size(); ++i) {
                        run += probs[i];
                        if (uu < run) {
                            pick = i;
                            break;
                        }
                    }
                    const double pp = probs[pick], sc = 1.0 / std::sqrt(pp);
                    const double* K = kraus + 32 * (size_t)(k0 + pick);
                    for (int a = 0; a < D; ++a)
                        for (int i = 0; i < D; ++i)
                            km[(size_t)b * D * D + a * D + i] =
                                make_double2(K[(a * 4 + i) * 2] * sc, K[(a * 4 + i) * 2 + 1] * sc);
                    logp[b] += std::log(pp / acc) + std::log(acc);
                }
                QF_CUDA(cudaMemcpyAsync(d_k.p, km.data(), (size_t)nb * D * D * 16, cudaMemcpyHostToDevice, s));
                QF_CUDA(launch_apply_local(precision, ctx->lam.p, n, nb, P0[j], P1[j], (const double2*)d_k.p, true, s));
                ctx->launches += 2;
            }
        }
        if (log_probs)
            for (int b = 0; b < nb; ++b) log_probs[t0 + b] = logp[b];
        if (obs) {
            HArgs ha{};
            ha.psi = ctx->lam.p;
            ha.n = n;
            ha.kh = od->plan.kh;
            ha.groups = (const DevGroup*)od->groups.p;
            ha.n_groups = (int)od->plan.groups.size();
            ha.terms = (const DevTerm*)od->terms.p;
            ha.write_lam = 0;
            ha.epart = (double*)d_part.p;
            QF_CUDA(launch_hpsi(precision, ha, nb, s));
            ReduceArgs ra{};
            ra.part = (const double*)d_part.p;
            ra.count = 1;
            ra.tiles = tiles_h;
            ra.out = (double*)d_E.p;
            QF_CUDA(launch_reduce(ra, nb, s));
            QF_CUDA(cudaMemcpyAsync(expvals + t0, d_E.p, (size_t)nb * 8, cudaMemcpyDeviceToHost, s));
        }
        if (states) {
            if (precision == QF_C128) {
                QF_CUDA(cudaMemcpyAsync(states + (size_t)t0 * 2 * N, ctx->lam.p, (size_t)nb * N * 16,
                                        cudaMemcpyDeviceToHost, s));
            } else {
                fbuf.resize((size_t)nb * 2 * N);
                QF_CUDA(cudaMemcpyAsync(fbuf.data(), ctx->lam.p, (size_t)nb * N * 8, cudaMemcpyDeviceToHost, s));
                QF_CUDA(cudaStreamSynchronize(s));
                for (size_t i = 0; i < fbuf.size(); ++i) states[(size_t)t0 * 2 * N + i] = fbuf[i];
            }
        }
        QF_CUDA(cudaStreamSynchronize(s));
    }
    return QF_OK;
}

int qf_ctx_set_timing(qf_ctx* ctx, int enabled) {
    if (!ctx) return set_err(QF_EINVAL, "null context");
    ctx->timing = enabled != 0;
    return QF_OK;
}

int qf_ctx_reset_stats(qf_ctx* ctx) {
    if (!ctx) return set_err(QF_EINVAL, "null context");
    reset_stats(ctx);
    return QF_OK;
}

int qf_ctx_stats(qf_ctx* ctx, long long* launches, long long* class_launches, double* ms, double* bytes) {
    if (!ctx) return set_err(QF_EINVAL, "null context");
    resolve_events(ctx);
    if (launches) *launches = ctx->launches;
    for (int i = 0; i < 4; ++i)
        if (class_launches) class_launches[i] = ctx->class_launches[i];
    for (int i = 0; i < 4; ++i) {
        if (ms) ms[i] = ctx->ms[i];
        if (bytes) bytes[i] = ctx->bytes[i];
    }
    return QF_OK;
}

}  // extern "C"
