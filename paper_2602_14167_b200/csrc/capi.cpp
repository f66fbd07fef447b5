// capi.cpp -- the C-ABI (include/qforge_b200.h): contexts, compiled programs and
// observables, chunked batch evaluation, NCCL sharding.
//
// Evaluation of one batch chunk (all on the context stream, no host sync):
//   forward sweeps (fused tile kernels) -> H|psi> + energy partials ->
//   adjoint sweeps with gradient taps -> fixed-order reductions.
// The reference evaluates 1 + 2P full energies per gradient
// (src/variational.cpp:54-81); this evaluates one forward and one adjoint pass.
#include "capi_internal.hpp"

#include <unistd.h>

namespace qfcapi {

NcclApi g_nccl;
std::mutex g_nccl_mu;

}  // namespace qfcapi

namespace qfcapi {

// Drops the context's captured evaluation graph (it may reference kernels,
// plans or buffers that are about to be released or rebuilt).
void drop_graph(qf_ctx* ctx) {
    if (ctx->graph_exec) {
        cudaStreamSynchronize(ctx->stream);
        cudaGraphExecDestroy(ctx->graph_exec);
        ctx->graph_exec = nullptr;
    }
    ctx->graph_key.clear();
    ctx->graph_nocapture_key.clear();
}

int ensure_obs_dev(qf_observable* o, int prec, int kh, ObsDev& d, int t_begin, int t_end) {
    if (d.ready && d.plan.kh == kh) return QF_OK;
    if (d.hj.kernel) {  // the previous plan's specialised kernel goes with it
        drop_graph(o->ctx);
        jit_release(d.hj);
    }
    std::string e = build_observable_plan(o->n, t_end - t_begin, o->codes.data() + (size_t)t_begin * o->n,
                                          o->w_re.data() + t_begin, o->w_im.data() + t_begin, kh, d.plan);
    if (!e.empty()) return set_err(QF_EINVAL, e);
    cudaStream_t s = o->ctx->stream;
    QF_CUDA(upload(d.groups, d.plan.groups, s));
    QF_CUDA(upload(d.terms, d.plan.terms, s));
    d.ready = true;
    d.hj_state = 0;  // plan (re)built: the specialised H|psi> kernel follows it
    static std::atomic<uint64_t> next_gen{1};
    d.gen = next_gen++;  // captured graphs of the previous plan (its kernel, groups, terms) are stale
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
        cudaEventElapsedTime(&ms, ctx->ev_pool[pr.start], ctx->ev_pool[pr.end]);
        if (pr.cls < 4) {
            ctx->ms[pr.cls] += ms;
        } else {  // per-launch timing (timing level 2): id = class - 100
            auto& e = ctx->launch_ms[pr.cls - 100];
            e.first += ms;
            e.second += 1;
        }
    }
    ctx->pending.clear();
    ctx->ev_used = 0;
}

// records an event on s (the pool is recycled only between evaluations, when
// every pending pair is complete: see resolve_events calls)
size_t record_event(qf_ctx* ctx, cudaStream_t s) {
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
            const size_t end = record_event(ctx, s);
            ctx->pending.push_back({ev_start[i / 2], end, cls});
        }
    };
    // timing level 2: every sweep / H|psi> launch bracketed by its own events
    // (ids: forward sweep i, 1000 = H|psi>, 2000 + i = adjoint sweep i)
    size_t l_ev = 0;
    auto ltick = [&] {
        if (ctx->timing >= 2) l_ev = record_event(ctx, s);
    };
    auto ltock = [&](int id) {
        if (ctx->timing >= 2) {
            const size_t end = record_event(ctx, s);
            ctx->pending.push_back({l_ev, end, 100 + id});
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
        ltick();
        if (prog->use_jit)
            QF_CUDA((cudaError_t)jit_launch(prog->jf.sweeps[i], sa, 1 << (n - sa.sw.k), bc, s));
        else
            QF_CUDA(launch_sweep(prec, false, sa, bc, P.fwd.max_mat, 0, s));
        ltock((int)i);
        ctx->launches++;
        ctx->class_launches[0]++;
        ctx->bytes[0] += (double)bc * N * vs * (sa.from_zero ? 1 : 2);
        ctx->flops[0] += (double)bc * N * prog->fwd_fpa[i];
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
    ha.prefetch = od->plan.terms.size() <= 4 * std::max<size_t>(1, od->plan.groups.size()) ? 1 : 0;
    static const bool hpsi_tma = !(std::getenv("QF_HPSI_TMA") && std::getenv("QF_HPSI_TMA")[0] == '0');
    ha.tma = hpsi_tma ? 1 : 0;
    ltick();
    if (od->hj_state == 1)
        QF_CUDA((cudaError_t)jit_launch_hpsi(od->hj, ha, tiles_h, bc, s));
    else
        QF_CUDA(launch_hpsi(prec, ha, bc, s));
    ltock(1000);
    ctx->launches++;
    ctx->class_launches[1]++;
    // compulsory bytes: psi read once, lambda written once (partner tiles of
    // flips above the tile are re-reads, served from L2 when the state fits)
    ctx->bytes[1] += (double)bc * N * vs * (grads ? 2 : 1);
    ctx->flops[1] += (double)bc * N * 4.0 * ((double)od->plan.terms.size() + 1.0);  // one real-weighted complex FMA per term
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
        if (const char* e = std::getenv("QF_DEV_BWD_PAUSE_US")) {  // development: idle GPU before the adjoint
            cudaStreamSynchronize(s);
            usleep((useconds_t)std::atol(e));
        }
        tick(4);
        const int nt = P.bwd.n_taps;
        const int tiles_b = 1 << (n - P.bwd.k);
        sa.phases = (const DevPhase*)prog->bwd.phases.p;
        sa.ops = (const DevOp*)prog->bwd.ops.p;
        sa.from_zero = 0;
        sa.tap_part = (double*)ctx->tap_part.p;
        sa.n_taps_total = nt;
        sa.gmat_pass_base = P.fwd.total_mat;
        // development: QF_DEBUG_BWD_STOP=i leaves psi/lambda as the first i adjoint sweeps left them
        size_t bwd_stop = P.bwd.sweeps.size();
        if (const char* e = std::getenv("QF_DEBUG_BWD_STOP")) bwd_stop = std::min(bwd_stop, (size_t)std::atol(e));
        for (size_t i = 0; i < bwd_stop; ++i) {
            sa.sw = P.bwd.sweeps[i];
            ltick();
            if (prog->use_jit)
                QF_CUDA((cudaError_t)jit_launch(prog->jb.sweeps[i], sa, 1 << (n - sa.sw.k), bc, s));
            else
                QF_CUDA(launch_sweep(prec, true, sa, bc, P.bwd.max_mat, P.bwd.max_taps, s));
            ltock(2000 + (int)i);
            ctx->launches++;
            ctx->class_launches[2]++;
            ctx->bytes[2] += (double)bc * N * vs * 4;
            ctx->flops[2] += (double)bc * N * prog->bwd_fpa[i];
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

// Resolve the observable's specialised H|psi> kernel (compiled at most once;
// outside any stream capture).
void ensure_hpsi_kernel(qf_program* prog, ObsDev* od, int prec) {
    if (prog->use_jit && od->hj_state == 0 && !(std::getenv("QF_JIT_HPSI") && std::getenv("QF_JIT_HPSI")[0] == '0')) {
        std::string err;
        od->hj_state = ((int)od->plan.terms.size() <= kJitHpsiMaxTerms && jit_build_hpsi(od->plan, prec, od->hj, err))
                           ? 1 : -1;
    }
    if (!prog->use_jit && od->hj_state == 0) od->hj_state = -1;
}

// Evaluate rows [0, batch) of device thetas into device outputs (chunked).
int eval_device(qf_ctx* ctx, qf_program* prog, qf_observable* obs, int batch, const double* d_thetas,
                double* d_E, double* d_Eim, double* d_G, bool term_shard, int rank, int world) {
    const ProgramPlan& P = prog->plan;
    if (obs->n != P.n) return set_err(QF_EINVAL, "expectation_pauli: size mismatch");
    if (d_G && !P.adjoint_ok) return set_err(QF_EINVAL, P.adjoint_error);
    const int prec = P.prec, n = P.n;
    const Geometry geo = geometry(prec, n);
    ObsDev* od = &obs->dev[prec];
    if (ctx->timing && ctx->ev_used > 4096) resolve_events(ctx);  // recycle the event pool between calls
    int rc;
    if (term_shard && world > 1) {
        // rank r owns the contiguous term block [T r / p, T (r + 1) / p)
        int64_t t0 = 0, t1 = 0;
        qf_shard_range((int64_t)obs->w_re.size(), rank, world, &t0, &t1);
        if (obs->shard_world != world || obs->shard_rank != rank) {
            obs->shard_dev[0].ready = obs->shard_dev[1].ready = false;
            obs->shard_world = world;
            obs->shard_rank = rank;
        }
        od = &obs->shard_dev[prec];
        rc = ensure_obs_dev(obs, prec, geo.kh, *od, (int)t0, (int)t1);
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
    // The work buffers already hold the whole batch (a repeated call): one
    // chunk, no device memory query (cudaMemGetInfo costs more than a small
    // state's whole evaluation).
    const size_t whole = (size_t)batch * N * vs;
    const bool resident = !budget && batch <= 65535 && ctx->psi.cap >= whole &&
                          (!grads || (ctx->lam.cap >= whole && ctx->tap_part.cap >= (size_t)batch * nt * tiles_b * 8 &&
                                      ctx->tapsum.cap >= (size_t)batch * nt * 8)) &&
                          ctx->epart.cap >= (size_t)batch * tiles_h * 8 &&
                          ctx->gmat.cap >= (size_t)batch * (P.fwd.total_mat + P.bwd.total_mat) * vs;
    if (resident) budget = per_entry * (size_t)batch;
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
    ensure_hpsi_kernel(prog, od, prec);
    // Single-chunk evaluations (small states / batches are launch bound) run as a
    // CUDA graph: captured on first use, replayed while everything it captured is
    // unchanged (program and observable identity, plan buffers, work buffers,
    // argument pointers, batch).
    static const bool graphs_off = std::getenv("QF_GRAPHS") && std::getenv("QF_GRAPHS")[0] == '0';
    if (bc >= batch && !ctx->timing && !graphs_off) {
        const std::vector<const void*> key = {
            (const void*)prog->uid, (const void*)obs->uid, (const void*)od->gen, od, od->groups.p, od->terms.p,
            (const void*)(intptr_t)od->hj_state, od->hj.kernel,
            od_im, (const void*)(intptr_t)batch, d_thetas, d_E, d_Eim, d_G, ctx->psi.p, ctx->lam.p, ctx->tap_part.p,
            ctx->tapsum.p, ctx->epart.p, ctx->gmat.p, ctx->zero_init.p, prog->init.p};
        if (ctx->graph_exec && key == ctx->graph_key) {
            QF_CUDA(cudaGraphLaunch(ctx->graph_exec, ctx->stream));
            ctx->launches += ctx->graph_launches;
            return QF_OK;
        }
        if (key != ctx->graph_nocapture_key) {
            const long long l0 = ctx->launches;
            QF_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            rc = eval_chunk(ctx, prog, od, 0, batch, d_thetas, d_E, d_Eim, d_G, od_im);
            cudaGraph_t g = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &g);
            cudaGraphExec_t exec = nullptr;
            if (!rc && ce == cudaSuccess && g && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) {
                cudaGraphDestroy(g);
                if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
                ctx->graph_exec = exec;
                ctx->graph_key = key;
                ctx->graph_launches = ctx->launches - l0;
                QF_CUDA(cudaGraphLaunch(ctx->graph_exec, ctx->stream));
                return QF_OK;
            }
            // not capturable here: run uncaptured (and do not retry this configuration)
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            ctx->launches = l0;
            ctx->graph_nocapture_key = key;
        }
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

int stage_thetas(qf_ctx* ctx, const qf_program* prog, int batch, const double* thetas) {
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
int forward_one(qf_ctx* ctx, qf_program* prog, const double* d_theta) {
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

}  // namespace qfcapi

extern "C" {

int qf_abi_version(void) { return QF_ABI_VERSION; }

int qf_shard_range(int64_t count, int rank, int world, int64_t* begin, int64_t* end) {
    if (!begin || !end || world < 1 || rank < 0 || rank >= world || count < 0)
        return set_err(QF_EINVAL, "qf_shard_range: bad arguments");
    *begin = count * rank / world;
    *end = count * (rank + 1) / world;
    return QF_OK;
}
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
    for (auto& kv : c->noise_progs) qf_program_destroy(kv.second);
    for (DevBuf* b : {&c->psi, &c->lam, &c->tap_part, &c->tapsum, &c->epart, &c->thetas, &c->out, &c->zero_init,
                      &c->gmat, &c->ul_state, &c->ul_aux, &c->coo_off, &c->coo_scratch, &c->coo_groups, &c->coo_terms, &c->coo_nodes, &c->coo_rows,
                      &c->coo_cols, &c->coo_vals})
        b->release();
    c->pin.release();
    for (auto& ev : c->ev_pool) cudaEventDestroy(ev);
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
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
    // minimal algorithmic flops per amplitude of every sweep, FMA
    // = 2: 6 per real rotation (ry, rx, h: two real products and a sum per
    // component), 14 per dense complex one-qubit gate, 6 per diagonal phase (one
    // complex product), 30 per dense 4x4 (per amplitude share), 0 for
    // permutations (x, cx); the adjoint applies each gate to two states and adds
    // 4 per gradient-tap product (one component of conj(lambda) G psi + the sum)
    for (int pi = 0; pi < 2; ++pi) {
        const PassPlan& pp = pi ? p->plan.bwd : p->plan.fwd;
        std::vector<double>& out = pi ? p->bwd_fpa : p->fwd_fpa;
        for (const DevSweep& sw : pp.sweeps) {
            double f = 0;
            for (int o = sw.op_begin; o < sw.op_end; ++o) {
                switch (pp.ops[o].kind) {
                    case DK_G1: f += 14.0 * (pi ? 2 : 1); break;
                    case DK_R1: case DK_RX: case DK_RS: f += 6.0 * (pi ? 2 : 1); break;
                    case DK_D1: case DK_D2: f += 6.0 * (pi ? 2 : 1); break;
                    case DK_G2: f += 30.0 * (pi ? 2 : 1); break;
                    case DK_TX: case DK_TY: case DK_TZ: case DK_TZZ: f += 4.0; break;
                    default: break;
                }
            }
            out.push_back(f);
        }
    }
    const char* jit_env = std::getenv("QF_JIT");
    if (!(jit_env && jit_env[0] == '0') && !p->plan.gates.empty()) {
        p->use_jit = jit_build(p->plan, p->jf, p->jb, p->jst);
        if (!p->use_jit && jit_env && jit_env[0] == '2') {  // QF_JIT=2: specialised kernels required
            std::string why = p->jst.error;
            delete p;
            return set_err(QF_ERUNTIME, "JIT required but unavailable: " + why);
        }
    }
    static std::atomic<uint64_t> next_prog_uid{1};
    p->uid = next_prog_uid++;
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
    if (!p->ctx->graph_key.empty() && p->ctx->graph_key[0] == (const void*)p->uid) drop_graph(p->ctx);
    jit_release(p->jf.sweeps);  // unload its modules (shared ones stay loaded for their other users)
    jit_release(p->jb.sweeps);
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
    // the program-creation compile stage (parallel, disk cache, out-of-process
    // NVRTC helper) without loading modules: works on a host without a GPU
    JitPass f, b;
    JitStats st;
    if (!jit_build(P, f, b, st, false)) return set_err(QF_ERUNTIME, st.error);
    if (kernels) *kernels = (int)(P.fwd.sweeps.size() + P.bwd.sweeps.size());
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

int qf_debug_copy_state(qf_ctx* ctx, int which, void* dst, size_t bytes) {
    if (!ctx || !dst) return set_err(QF_EINVAL, "qf_debug_copy_state: bad arguments");
    const DevBuf& b = which ? ctx->lam : ctx->psi;
    if (bytes > b.cap) return set_err(QF_EINVAL, "qf_debug_copy_state: more bytes than the buffer holds");
    QF_CUDA(cudaSetDevice(ctx->device));
    QF_CUDA(cudaStreamSynchronize((cudaStream_t)ctx->stream));
    QF_CUDA(cudaMemcpy(dst, b.p, bytes, cudaMemcpyDefault));
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
    if (o->ctx->graph_key.size() > 1 && o->ctx->graph_key[1] == (const void*)o->uid) drop_graph(o->ctx);
    for (auto* d : {&o->dev[0], &o->dev[1], &o->shard_dev[0], &o->shard_dev[1]}) {
        jit_release(d->hj);
        d->groups.release();
        d->terms.release();
    }
    delete o;
    return QF_OK;
}

static void reset_stats(qf_ctx* ctx) {
    resolve_events(ctx);
    ctx->launches = 0;
    for (int i = 0; i < 4; ++i) {
        ctx->ms[i] = ctx->bytes[i] = ctx->flops[i] = 0;
        ctx->class_launches[i] = 0;
    }
    ctx->launch_ms.clear();
}

}  // extern "C"

namespace qfcapi {

// The contribution of `rank` of `world` to a batched evaluation, written into
// the zero-padded [batch x (1 + P)] float64 device buffer d_out (energies, then
// gradients): batch sharding evaluates rows [B r / p, B (r + 1) / p) and leaves
// the other rows 0 (so the sum over ranks is exact: x + 0 = x); term sharding
// evaluates every row on the rank's term block (energy and gradient are linear
// in H).  The NCCL path all-reduces exactly this buffer.
int eval_shard(qf_ctx* ctx, qf_program* prog, qf_observable* obs, int batch, const double* d_thetas, int rank,
               int world, bool grads, double* d_out) {
    const int P = prog->plan.n_params;
    double* dE = d_out;
    double* dG = grads ? d_out + batch : nullptr;
    if (world > 1 && obs->term_shard)
        return eval_device(ctx, prog, obs, batch, d_thetas, dE, nullptr, dG, true, rank, world);
    int64_t b0 = 0, b1 = 0;
    qf_shard_range(batch, rank, world, &b0, &b1);
    if (world > 1)
        QF_CUDA(cudaMemsetAsync(d_out, 0, (size_t)batch * (1 + (grads ? P : 0)) * 8, ctx->stream));
    if (b1 <= b0) return QF_OK;
    return eval_device(ctx, prog, obs, (int)(b1 - b0), d_thetas + (size_t)b0 * P, dE + b0, nullptr,
                       dG ? dG + (size_t)b0 * P : nullptr, false, 0, 1);
}

int allreduce_out(qf_ctx* ctx, double* d_out, size_t count) {
    const int r = g_nccl.allReduce(d_out, d_out, count, kNcclFloat64, kNcclSum, ctx->comm, ctx->stream);
    if (r) return set_err(QF_ENCCL, std::string("ncclAllReduce: ") + g_nccl.errStr(r));
    return QF_OK;
}

// host-buffer evaluation of one (virtual) rank's share; collective when requested
int eval_host(qf_ctx* ctx, qf_program* prog, qf_observable* obs, int batch, const double* thetas, int rank,
              int world, bool collective, double* energies, double* grads) {
    if (grads && !prog->plan.adjoint_ok) return set_err(QF_EINVAL, prog->plan.adjoint_error);
    int rc = check_thetas(prog, batch, thetas);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    const int P = prog->plan.n_params;
    rc = stage_thetas(ctx, prog, batch, thetas);
    if (rc) return rc;
    const size_t out_n = (size_t)batch * (1 + (grads ? P : 0));
    QF_CUDA(ctx->out.reserve(out_n * 8));
    double* d_out = (double*)ctx->out.p;
    rc = eval_shard(ctx, prog, obs, batch, (const double*)ctx->thetas.p, rank, world, grads != nullptr, d_out);
    if (rc) return rc;
    if (collective) {
        rc = allreduce_out(ctx, d_out, out_n);
        if (rc) return rc;
    }
    QF_CUDA(ctx->pin.reserve(out_n * 8));
    QF_CUDA(cudaMemcpyAsync(ctx->pin.p, d_out, out_n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    QF_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(energies, ctx->pin.p, (size_t)batch * 8);
    if (grads) std::memcpy(grads, (double*)ctx->pin.p + batch, (size_t)batch * P * 8);
    return QF_OK;
}

}  // namespace qfcapi

extern "C" {

int qf_energy_grad_batch(qf_ctx* ctx, const qf_program* cprog, const qf_observable* cobs, int batch,
                         const double* thetas, double* energies, double* grads) {
    qf_program* prog = const_cast<qf_program*>(cprog);
    qf_observable* obs = const_cast<qf_observable*>(cobs);
    if (!ctx || !prog || !obs || batch < 0 || (batch > 0 && (!energies || (!thetas && prog->plan.n_params))))
        return set_err(QF_EINVAL, "qf_energy_grad_batch: bad arguments");
    if (batch == 0) return QF_OK;
    const bool sharded = ctx->comm != nullptr;
    return eval_host(ctx, prog, obs, batch, thetas, sharded ? ctx->rank : 0, sharded ? ctx->world : 1, sharded,
                     energies, grads);
}

int qf_energy_grad_batch_partial(qf_ctx* ctx, const qf_program* cprog, const qf_observable* cobs, int batch,
                                 const double* thetas, int rank, int world, double* energies, double* grads) {
    qf_program* prog = const_cast<qf_program*>(cprog);
    qf_observable* obs = const_cast<qf_observable*>(cobs);
    if (!ctx || !prog || !obs || batch < 0 || world < 1 || rank < 0 || rank >= world ||
        (batch > 0 && (!energies || (!thetas && prog->plan.n_params))))
        return set_err(QF_EINVAL, "qf_energy_grad_batch_partial: bad arguments");
    if (batch == 0) return QF_OK;
    return eval_host(ctx, prog, obs, batch, thetas, rank, world, false, energies, grads);
}

}  // extern "C"

namespace qfcapi {

// device-buffer evaluation with the context's sharding (stream-ordered)
int eval_entry_device(qf_ctx* ctx, qf_program* prog, qf_observable* obs, int batch, const double* d_thetas,
                      double* d_energies, double* d_grads) {
    if (!ctx->comm)
        return eval_device(ctx, prog, obs, batch, d_thetas, d_energies, nullptr, d_grads, false, 0, 1);
    // sharded: the rank's share into the zero-padded buffer, one all-reduce, then
    // the caller's buffers (stream-ordered; no host sync)
    const int P = prog->plan.n_params;
    const size_t out_n = (size_t)batch * (1 + (d_grads ? P : 0));
    QF_CUDA(ctx->out.reserve(out_n * 8));
    double* d_out = (double*)ctx->out.p;
    int rc = eval_shard(ctx, prog, obs, batch, d_thetas, ctx->rank, ctx->world, d_grads != nullptr, d_out);
    if (rc) return rc;
    rc = allreduce_out(ctx, d_out, out_n);
    if (rc) return rc;
    QF_CUDA(cudaMemcpyAsync(d_energies, d_out, (size_t)batch * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    if (d_grads)
        QF_CUDA(cudaMemcpyAsync(d_grads, d_out + batch, (size_t)batch * P * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return QF_OK;
}

}  // namespace qfcapi

extern "C" {

int qf_energy_grad_batch_device(qf_ctx* ctx, const qf_program* cprog, const qf_observable* cobs, int batch,
                                const double* d_thetas, double* d_energies, double* d_grads) {
    qf_program* prog = const_cast<qf_program*>(cprog);
    qf_observable* obs = const_cast<qf_observable*>(cobs);
    if (!ctx || !prog || !obs || batch < 0 || (batch > 0 && !d_energies))
        return set_err(QF_EINVAL, "qf_energy_grad_batch_device: bad arguments");
    if (batch == 0) return QF_OK;
    cudaSetDevice(ctx->device);
    return eval_entry_device(ctx, prog, obs, batch, d_thetas, d_energies, d_grads);
}

int qf_vqe_run(qf_ctx* ctx, const qf_program* cprog, const qf_observable* cobs, int batch, const double* theta0,
               int steps, double lr, int grad_mode, double fd_step, double* traces, double* final_thetas,
               double* best_energy, int* best_index) {
    // vqe_run (reference src/variational.cpp:103-143) with the whole batch resident:
    // per step one batched energy (+ adjoint gradient, or one batched call over the
    // 2P shifted parameter sets) and one Adam kernel; one host copy at the end.
    qf_program* prog = const_cast<qf_program*>(cprog);
    qf_observable* obs = const_cast<qf_observable*>(cobs);
    if (!ctx || !prog || !obs || !theta0 || !traces || !final_thetas || !best_energy || !best_index)
        return set_err(QF_EINVAL, "qf_vqe_run: null argument");
    if (batch < 1) return set_err(QF_EINVAL, "vqe_run: empty batch");
    if (steps < 1) return set_err(QF_EINVAL, "vqe_run: steps must be >= 1");
    if (grad_mode < QF_GRAD_PARAMETER_SHIFT || grad_mode > QF_GRAD_ADJOINT)
        return set_err(QF_EINVAL, "qf_vqe_run: bad gradient mode");
    if (grad_mode == QF_GRAD_FINITE_DIFF && !(fd_step > 0.0))
        return set_err(QF_EINVAL, "gradient: finite-diff step must be positive");
    const int P = prog->plan.n_params;
    if (grad_mode == QF_GRAD_ADJOINT && !prog->plan.adjoint_ok) return set_err(QF_EINVAL, prog->plan.adjoint_error);
    if (grad_mode == QF_GRAD_PARAMETER_SHIFT)
        for (const auto& gi : prog->plan.gates)
            if (gi.g.slot >= 0 && !gi.gen)
                return set_err(QF_EINVAL, "gradient: parameter not shift-eligible, use finite_diff");
    int rc = check_thetas(prog, batch, theta0);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const size_t BP = (size_t)batch * P;
    LocalBuf th, m, v, g, tr, sh, es;
    QF_CUDA(th.reserve(std::max<size_t>(16, BP * 8)));
    QF_CUDA(m.reserve(std::max<size_t>(16, BP * 8)));
    QF_CUDA(v.reserve(std::max<size_t>(16, BP * 8)));
    QF_CUDA(g.reserve(std::max<size_t>(16, BP * 8)));
    QF_CUDA(tr.reserve((size_t)(steps + 1) * batch * 8));
    QF_CUDA(cudaMemsetAsync(m.p, 0, std::max<size_t>(16, BP * 8), s));
    QF_CUDA(cudaMemsetAsync(v.p, 0, std::max<size_t>(16, BP * 8), s));
    QF_CUDA(cudaMemsetAsync(g.p, 0, std::max<size_t>(16, BP * 8), s));
    if (BP) QF_CUDA(cudaMemcpyAsync(th.p, theta0, BP * 8, cudaMemcpyHostToDevice, s));
    const bool shifted = grad_mode != QF_GRAD_ADJOINT && P > 0;
    const double shift = grad_mode == QF_GRAD_PARAMETER_SHIFT ? M_PI / 2.0 : fd_step;
    const double denom = grad_mode == QF_GRAD_PARAMETER_SHIFT ? 2.0 : 2.0 * fd_step;
    if (shifted) {
        QF_CUDA(sh.reserve(BP * 2 * P * 8));
        QF_CUDA(es.reserve(BP * 2 * 8));
    }
    double* d_th = (double*)th.p;
    double* d_tr = (double*)tr.p;
    for (int st = 0; st < steps; ++st) {
        double* d_e = d_tr + (size_t)st * batch;
        if (grad_mode == QF_GRAD_ADJOINT) {
            rc = eval_entry_device(ctx, prog, obs, batch, d_th, d_e, (double*)g.p);
        } else {
            rc = eval_entry_device(ctx, prog, obs, batch, d_th, d_e, nullptr);
            if (!rc && shifted) {
                QF_CUDA(launch_shift_thetas(batch, P, d_th, shift, (double*)sh.p, s));
                rc = eval_entry_device(ctx, prog, obs, (int)(2 * BP), (const double*)sh.p, (double*)es.p, nullptr);
                if (!rc) QF_CUDA(launch_shift_grad(batch, P, (const double*)es.p, denom, (double*)g.p, s));
            }
        }
        if (rc) return rc;
        const double c1 = 1.0 - std::pow(0.9, st + 1), c2 = 1.0 - std::pow(0.999, st + 1);
        QF_CUDA(launch_adam((int)BP, d_th, (double*)m.p, (double*)v.p, (const double*)g.p, lr, 0.9, 0.999, 1e-8,
                            c1, c2, s));
        ctx->launches += 1 + (shifted ? 2 : 0);
    }
    rc = eval_entry_device(ctx, prog, obs, batch, d_th, d_tr + (size_t)steps * batch, nullptr);
    if (rc) return rc;
    std::vector<double> trh((size_t)(steps + 1) * batch);
    QF_CUDA(cudaMemcpyAsync(trh.data(), d_tr, trh.size() * 8, cudaMemcpyDeviceToHost, s));
    if (BP) QF_CUDA(cudaMemcpyAsync(final_thetas, d_th, BP * 8, cudaMemcpyDeviceToHost, s));
    QF_CUDA(cudaStreamSynchronize(s));
    *best_energy = INFINITY;
    *best_index = -1;
    for (int b = 0; b < batch; ++b) {
        for (int st = 0; st <= steps; ++st) traces[(size_t)b * (steps + 1) + st] = trh[(size_t)st * batch + b];
        if (trh[(size_t)steps * batch + b] < *best_energy) {  // strict <, first index wins (:133-141)
            *best_energy = trh[(size_t)steps * batch + b];
            *best_index = b;
        }
    }
    return QF_OK;
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
    rc = eval_device(ctx, prog, obs, 1, (const double*)ctx->thetas.p, dE, dE + 1, nullptr, false, 0, 1);
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

int qf_ctx_set_timing(qf_ctx* ctx, int enabled) {
    if (!ctx) return set_err(QF_EINVAL, "null context");
    ctx->timing = enabled < 0 ? 0 : enabled;
    return QF_OK;
}

int qf_ctx_flops(qf_ctx* ctx, double* flops_by_class) {
    if (!ctx || !flops_by_class) return set_err(QF_EINVAL, "qf_ctx_flops: bad arguments");
    for (int i = 0; i < 4; ++i) flops_by_class[i] = ctx->flops[i];
    return QF_OK;
}

int qf_ctx_launch_times(qf_ctx* ctx, int cap, int* ids, double* ms, long long* counts, int* n) {
    if (!ctx || !n || cap < 0) return set_err(QF_EINVAL, "qf_ctx_launch_times: bad arguments");
    resolve_events(ctx);
    int k = 0;
    for (const auto& kv : ctx->launch_ms) {
        if (k < cap) {
            if (ids) ids[k] = kv.first;
            if (ms) ms[k] = kv.second.first;
            if (counts) counts[k] = kv.second.second;
        }
        ++k;
    }
    *n = k;
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
