// capi_traj.cpp -- the trajectory workloads of the C-ABI:
// MIPT-Haar (qf_mipt_haar), classical shadows (qf_shadow_snapshots) and Monte-Carlo
// noise trajectories (qf_noise_trajectories), on the batched sweep engine plus the
// measurement / sampling / local-operator kernels of traj.cu.
#include <cublas_v2.h>

#include <chrono>
#include <cstring>
#include <complex>
#include <thread>

#include "../../include/qforge/rng.hpp"
#include "capi_internal.hpp"

namespace {

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

// cuBLAS, loaded at run time: the batched ZGEMM that forms rho = A^H A for the
// trajectory entropy (the eigenvalues are our own kernels, eig.cu)
struct LinAlg {
    void* hb = nullptr;
    cublasHandle_t cb = nullptr;
    decltype(&cublasCreate_v2) bcreate = nullptr;
    decltype(&cublasSetStream_v2) bstream = nullptr;
    decltype(&cublasZgemmStridedBatched) zgemm_sb = nullptr;
    int device = -1;
    std::string err;
    bool load(int dev) {
        if (cb && device == dev) return true;
        if (!hb) {
            const char* bl[] = {"libcublas.so.12", "libcublas.so", "/usr/local/cuda/lib64/libcublas.so.12",
                                "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cublas/lib/libcublas.so.12"};
            for (const char* nm : bl)
                if ((hb = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
            if (!hb) {
                err = "cuBLAS unavailable (libcublas.so.12)";
                return false;
            }
            bcreate = (decltype(bcreate))dlsym(hb, "cublasCreate_v2");
            bstream = (decltype(bstream))dlsym(hb, "cublasSetStream_v2");
            zgemm_sb = (decltype(zgemm_sb))dlsym(hb, "cublasZgemmStridedBatched");
            if (!bcreate || !bstream || !zgemm_sb) {
                err = "cuBLAS lacks required symbols";
                return false;
            }
        }
        cb = nullptr;  // a handle belongs to the device current at creation
        if (bcreate(&cb) != CUBLAS_STATUS_SUCCESS) {
            err = "cublasCreate failed";
            return false;
        }
        device = dev;
        return true;
    }
};
LinAlg g_linalg;
std::mutex g_linalg_mu;

}  // namespace

extern "C" {

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
    std::lock_guard<std::mutex> linalg_lock(g_linalg_mu);  // the cuBLAS handle is process-wide
    if (!g_linalg.load(ctx->device)) return set_err(QF_ERUNTIME, g_linalg.err);
    LinAlg& la = g_linalg;
    // spectra in sub-batches: converted states (complex64) + rho + tridiagonals
    const size_t per_eig = (precision == QF_C64 ? N * 16 : 0) + (size_t)dk * dk * 16 + (size_t)dk * 16;
    // (one CTA per matrix, one CTA per SM: sub-batches are whole waves of the SM count)
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, ctx->device);
    size_t cap = ((size_t)6 << 30) / per_eig;
    if (cap > (size_t)n_sm) cap -= cap % (size_t)n_sm;
    const int esub = (int)std::max<size_t>(1, std::min<size_t>((size_t)bc, cap));
    LocalBuf d_conv, d_rho, d_tri;
    if (precision == QF_C64) QF_CUDA(d_conv.reserve((size_t)esub * N * 16));
    QF_CUDA(d_rho.reserve((size_t)esub * dk * dk * 16));
    QF_CUDA(d_tri.reserve((size_t)esub * dk * 16));
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
        // (double precision for both state precisions: a complex64 spectrum loses
        // the small Schmidt values, n = 20: -0.22 bits of mean entropy)
        if (la.bstream(la.cb, s) != CUBLAS_STATUS_SUCCESS) return set_err(QF_ERUNTIME, "cublasSetStream failed");
        for (int e0 = 0; e0 < nb; e0 += esub) {
            const int ne = std::min(esub, nb - e0);
            const cuDoubleComplex* A = (const cuDoubleComplex*)((const unsigned char*)ctx->psi.p + (size_t)e0 * N * vs);
            if (precision == QF_C64) {
                QF_CUDA(launch_convert_state(precision, A, (double*)d_conv.p, (int64_t)N * ne, s));
                A = (const cuDoubleComplex*)d_conv.p;
            }
            const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
            if (la.zgemm_sb(la.cb, CUBLAS_OP_C, CUBLAS_OP_N, (int)dk, (int)dk, (int)de, &one, A, (int)de,
                            (long long)N, A, (int)de, (long long)N, &zero, (cuDoubleComplex*)d_rho.p, (int)dk,
                            (long long)dk * dk, ne) != CUBLAS_STATUS_SUCCESS)
                return set_err(QF_ERUNTIME, "qf_mipt_haar: cuBLAS ZGEMM failed");
            QF_CUDA(launch_hermitian_eigvals((double2*)d_rho.p, (int)dk, ne, (double*)d_tri.p,
                                             (double*)d_tri.p + (size_t)ne * dk, (double*)d_w.p + (size_t)e0 * dk,
                                             s));
            ctx->launches += 3;
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

int qf_hermitian_eigvals(qf_ctx* ctx, int m, int batch, const double* a, double* w) {
    if (!ctx || m < 1 || m > 2048 || batch < 0 || (batch > 0 && (!a || !w)))
        return set_err(QF_EINVAL, "qf_hermitian_eigvals: bad arguments");
    if (batch == 0) return QF_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    LocalBuf d_a, d_t, d_w;
    const size_t mm = (size_t)m * m;
    QF_CUDA(d_a.reserve((size_t)batch * mm * 16));
    QF_CUDA(d_t.reserve((size_t)batch * m * 16));
    QF_CUDA(d_w.reserve((size_t)batch * m * 8));
    QF_CUDA(cudaMemcpyAsync(d_a.p, a, (size_t)batch * mm * 16, cudaMemcpyHostToDevice, s));
    QF_CUDA(launch_hermitian_eigvals((double2*)d_a.p, m, batch, (double*)d_t.p, (double*)d_t.p + (size_t)batch * m,
                                     (double*)d_w.p, s));
    ctx->launches += 2;
    QF_CUDA(cudaMemcpyAsync(w, d_w.p, (size_t)batch * m * 8, cudaMemcpyDeviceToHost, s));
    QF_CUDA(cudaStreamSynchronize(s));
    return QF_OK;
}

int qf_apply_unitary(qf_ctx* ctx, int n, double* state, int k, const int* wires, const double* u) {
    // reference circuit.cpp:78-176 (apply_local_unitary) on a host complex128 state:
    // one H2D copy, one kernel (no program, no JIT), one D2H copy
    if (!ctx || !state || !wires || !u || n < 1 || n > 30) return set_err(QF_EINVAL, "qf_apply_unitary: bad arguments");
    for (int i = 0; i < k; ++i)
        if (wires[i] < 0 || wires[i] >= n) return set_err(QF_EINVAL, "apply_local_unitary: wire out of range");
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < i; ++j)
            if (wires[i] == wires[j]) return set_err(QF_EINVAL, "apply_local_unitary: wires must be distinct");
    if (k < 1 || k > 13) return set_err(QF_EINVAL, "apply_local_unitary: 1 to 13 wires on the device path");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const size_t N = size_t(1) << n, DK = size_t(1) << k;
    QF_CUDA(ctx->ul_state.reserve(N * 16));
    QF_CUDA(ctx->ul_aux.reserve(64 + DK * DK * 16));
    int pos[13];
    for (int i = 0; i < k; ++i) pos[i] = n - 1 - wires[i];
    std::vector<double> buf(16 + DK * DK * 2, 0.0);
    std::memcpy(buf.data(), pos, sizeof(int) * k);
    double* um = buf.data() + 8;  // 64-byte header for the positions
    if (k <= 4) {
        std::memcpy(um, u, DK * DK * 16);
    } else {
        for (size_t i = 0; i < DK; ++i)  // column-major for the large-k kernel
            for (size_t j = 0; j < DK; ++j) {
                um[(j * DK + i) * 2] = u[(i * DK + j) * 2];
                um[(j * DK + i) * 2 + 1] = u[(i * DK + j) * 2 + 1];
            }
    }
    QF_CUDA(cudaMemcpyAsync(ctx->ul_aux.p, buf.data(), 64 + DK * DK * 16, cudaMemcpyHostToDevice, s));
    QF_CUDA(cudaMemcpyAsync(ctx->ul_state.p, state, N * 16, cudaMemcpyHostToDevice, s));
    const double2* dm = (const double2*)((const char*)ctx->ul_aux.p + 64);
    QF_CUDA(launch_apply_unitary((double2*)ctx->ul_state.p, n, k, (const int*)ctx->ul_aux.p, dm, dm, s));
    ctx->launches++;
    QF_CUDA(cudaMemcpyAsync(state, ctx->ul_state.p, N * 16, cudaMemcpyDeviceToHost, s));
    QF_CUDA(cudaStreamSynchronize(s));
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
    // Channel-free runs of >= 2 ops go through compiled fused-sweep programs (one
    // HBM pass per sweep instead of one per gate), cached on the context by content
    // (n, precision, ops, their matrices) so repeated calls reuse the kernels.
    struct Seg { int j0, j1; qf_program* prog; };
    std::vector<Seg> segs;
    size_t seg_mat = 16;
    if (ctx->noise_progs.size() > 256) {  // bound the cache (between calls, never inside one)
        QF_CUDA(cudaStreamSynchronize(s));
        for (auto& kv : ctx->noise_progs) qf_program_destroy(kv.second);
        ctx->noise_progs.clear();
    }
    for (int j = 0; j < n_ops;) {
        if (op_chan_ptr[j + 1] > op_chan_ptr[j]) { ++j; continue; }
        int j1 = j;
        while (j1 < n_ops && op_chan_ptr[j1 + 1] == op_chan_ptr[j1]) ++j1;
        if (j1 - j >= 2) {
            std::string key((const char*)&n, sizeof n);
            key.append((const char*)&precision, sizeof precision);
            for (int q = j; q < j1; ++q)  // every field but `reserved`
                key.append((const char*)(ops + q), offsetof(qf_op, reserved));
            for (int q = j; q < j1; ++q)
                if (ops[q].mat >= 0 && mats && ops[q].mat < n_mats)
                    key.append((const char*)(mats + 32 * (size_t)ops[q].mat), 32 * sizeof(double));
            qf_program*& pg = ctx->noise_progs[key];
            if (!pg) {
                int rc = qf_program_create(ctx, n, j1 - j, ops + j, mats, n_mats, 0, precision, &pg);
                if (rc) {
                    ctx->noise_progs.erase(key);
                    return rc;
                }
            }
            segs.push_back({j, j1, pg});
            seg_mat = std::max(seg_mat, (size_t)pg->plan.fwd.total_mat * vs);
        }
        j = j1;
    }
    if (!segs.empty()) QF_CUDA(ctx->gmat.reserve((size_t)bc * seg_mat));
    // Kraus operators, uniforms, log-probabilities and the error flag live on the
    // device: branch picks run in a kernel, so a chunk needs no host round trip
    // until its results are read back.
    LocalBuf d_kraus, d_u, d_logp, d_err;
    const int n_kraus = n_apps > 0 ? chan_kraus_ptr[*std::max_element(op_chan, op_chan + n_apps) + 1] : 0;
    QF_CUDA(d_kraus.reserve(std::max<size_t>(16, (size_t)n_kraus * 32 * 8)));
    if (n_kraus) QF_CUDA(cudaMemcpyAsync(d_kraus.p, kraus, (size_t)n_kraus * 32 * 8, cudaMemcpyHostToDevice, s));
    QF_CUDA(d_u.reserve(std::max<size_t>(16, (size_t)bc * n_apps * 8)));
    QF_CUDA(d_logp.reserve((size_t)bc * 8));
    QF_CUDA(d_err.reserve(16));
    QF_CUDA(cudaMemsetAsync(d_err.p, 0, 4, s));
    std::vector<float> fbuf;
    for (int t0 = 0; t0 < trajectories; t0 += bc) {
        const int nb = std::min(bc, trajectories - t0);
        if (init)
            QF_CUDA(launch_init_state(precision, ctx->lam.p, d_init.p, n, nb, s));
        else
            QF_CUDA(launch_set_basis0(precision, ctx->lam.p, n, nb, s));
        QF_CUDA(cudaMemsetAsync(d_logp.p, 0, (size_t)nb * 8, s));
        if (n_apps)
            QF_CUDA(cudaMemcpyAsync(d_u.p, u + (size_t)t0 * n_apps, (size_t)nb * n_apps * 8, cudaMemcpyHostToDevice, s));
        int app = 0;
        size_t si = 0;
        // The last channel's branch K / sqrt(p) of an op stays pending in d_k and is
        // folded into the next noisy op's pass when their wires are disjoint
        // (apply2_rho: one state pass instead of two); otherwise it is applied alone.
        int pend = -1;
        auto flush = [&]() -> cudaError_t {
            if (pend < 0) return cudaSuccess;
            const cudaError_t e = launch_apply_local(precision, ctx->lam.p, n, nb, P0[pend], P1[pend],
                                                     (const double2*)d_k.p, true, s);
            ctx->launches++;
            pend = -1;
            return e;
        };
        auto disjoint = [&](int a, int b) {
            const uint32_t ma = (1u << P0[a]) | (P1[a] >= 0 ? 1u << P1[a] : 0u);
            const uint32_t mb = (1u << P0[b]) | (P1[b] >= 0 ? 1u << P1[b] : 0u);
            return (ma & mb) == 0;
        };
        static const bool fold = !(std::getenv("QF_NOISE_FOLD") && std::getenv("QF_NOISE_FOLD")[0] == '0');
        for (int j = 0; j < n_ops;) {
            if (si < segs.size() && segs[si].j0 == j) {  // fused channel-free run
                QF_CUDA(flush());
                qf_program* pg = segs[si].prog;
                const ProgramPlan& PP = pg->plan;
                SweepArgs sa{};
                sa.psi = ctx->lam.p;
                sa.n = n;
                sa.gates = (const DevGate*)pg->gates.p;
                sa.cmats = (const double*)pg->cmats.p;
                sa.gmat = ctx->gmat.p;
                sa.gmat_stride = PP.fwd.total_mat;
                QF_CUDA(launch_mats(precision, false, (const DevOp*)pg->fwd.ops.p, (const int*)pg->goff_fwd.p,
                                    (int)PP.fwd.ops.size(), sa.gates, sa.cmats, nullptr, 0, 0, ctx->gmat.p,
                                    sa.gmat_stride, 0, nb, s));
                sa.phases = (const DevPhase*)pg->fwd.phases.p;
                sa.ops = (const DevOp*)pg->fwd.ops.p;
                for (size_t i = 0; i < PP.fwd.sweeps.size(); ++i) {
                    sa.sw = PP.fwd.sweeps[i];
                    if (pg->use_jit)
                        QF_CUDA((cudaError_t)jit_launch(pg->jf.sweeps[i], sa, 1 << (n - sa.sw.k), nb, s));
                    else
                        QF_CUDA(launch_sweep(precision, false, sa, nb, PP.fwd.max_mat, 0, s));
                    ctx->launches++;
                }
                ctx->launches++;
                j = segs[si++].j1;
                continue;
            }
            const int c0 = op_chan_ptr[j], c1 = op_chan_ptr[j + 1];
            const double2* g = (const double2*)d_gm.p + (size_t)j * 16;
            if (c0 == c1) {
                QF_CUDA(flush());
                QF_CUDA(launch_apply_local(precision, ctx->lam.p, n, nb, P0[j], P1[j], g, false, s));
                ctx->launches++;
                ++j;
                continue;
            }
            // gate, then per channel: rho of the current state on the gate's wires ->
            // branch pick -> K / sqrt(p) (fused with the next channel's rho)
            if (fold && pend >= 0 && disjoint(pend, j)) {
                QF_CUDA(launch_apply2_rho(precision, ctx->lam.p, n, nb, P0[pend], P1[pend], (const double2*)d_k.p,
                                          P0[j], P1[j], g, (double2*)d_rho.p, s));
                pend = -1;
            } else {
                QF_CUDA(flush());
                QF_CUDA(launch_apply_rho(precision, ctx->lam.p, n, nb, P0[j], P1[j], g, false, (double2*)d_rho.p, s));
            }
            ctx->launches++;
            for (int ci = c0; ci < c1; ++ci, ++app) {
                const int ch = op_chan[ci];
                const int k0 = chan_kraus_ptr[ch], k1 = chan_kraus_ptr[ch + 1];
                if (k1 <= k0) return set_err(QF_EINVAL, "KrausChannel: no operators");
                QF_CUDA(launch_kraus_pick((const double2*)d_rho.p, parts, Dg[j], (const double*)d_kraus.p, k0, k1,
                                          (const double*)d_u.p, n_apps, app, (double2*)d_k.p, (double*)d_logp.p,
                                          (int*)d_err.p, nb, s));
                if (ci + 1 < c1) {
                    QF_CUDA(launch_apply_rho(precision, ctx->lam.p, n, nb, P0[j], P1[j], (const double2*)d_k.p, true,
                                             (double2*)d_rho.p, s));
                    ctx->launches += 2;
                } else {
                    pend = j;  // applied by the next pass (or flushed)
                    ctx->launches += 1;
                }
            }
            ++j;
        }
        QF_CUDA(flush());
        if (log_probs)
            QF_CUDA(cudaMemcpyAsync(log_probs + t0, d_logp.p, (size_t)nb * 8, cudaMemcpyDeviceToHost, s));
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
        int err = 0;
        QF_CUDA(cudaMemcpy(&err, d_err.p, 4, cudaMemcpyDeviceToHost));
        if (err) return set_err(QF_EINVAL, "mc_trajectory: all branch probabilities vanish");
    }
    return QF_OK;
}

}  // extern "C"
