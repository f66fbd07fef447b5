// capi_internal.hpp -- state shared by the C-ABI translation units (capi.cpp:
// contexts, programs, observables, batch evaluation, COO; capi_traj.cpp: the
// trajectory workloads).  Not part of the public interface.
#pragma once

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


#include "../../include/qforge_b200.h"
#include "kernels.cuh"
#include "jit.hpp"
#include "plan.hpp"


namespace qfcapi {

using namespace qfb;

inline thread_local std::string g_err;

inline int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

inline std::string launch_detail(const char* call) {
    return std::strstr(call, "jit_launch") ? " [" + qfb::jit_last_launch_detail() + "]" : std::string();
}


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
extern NcclApi g_nccl;
extern std::mutex g_nccl_mu;
constexpr int kNcclFloat64 = 8, kNcclSum = 0;


size_t vsize(int prec);

}  // namespace qfcapi

#define QF_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_err(QF_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                         " at " #call + launch_detail(#call));            \
    } while (0)

using namespace qfb;
using namespace qfcapi;

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
    uint64_t uid = 0;  // identity for the context's graph cache
    std::vector<double> fwd_fpa, bwd_fpa;  // canonical flops per amplitude of each sweep
};

struct ObsDev {
    ObservablePlan plan;
    DevBuf groups, terms;
    bool ready = false;
    JitKernel hj;       // specialised H|psi> kernel (jit.hpp)
    int hj_state = 0;   // 0 not built, 1 ready, -1 unavailable (AOT hpsi_kernel)
    uint64_t gen = 0;   // plan generation (process-unique; part of the graph-cache key)
};

struct qf_observable {
    qf_ctx* ctx = nullptr;
    int n = 0;
    std::vector<int8_t> codes;
    std::vector<double> w_re, w_im;
    ObsDev dev[2];         // per precision (tile bits differ)
    bool term_shard = false;
    int shard_world = 0, shard_rank = -1;  // term-sharded sub-plan cache key
    ObsDev shard_dev[2];
    uint64_t uid = 0;      // identity for the context's COO offset cache
};

struct qf_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    size_t budget = 0;
    DevBuf psi, lam, tap_part, tapsum, epart, thetas, out, zero_init, gmat;
    DevBuf ul_state, ul_aux;  // apply_local_unitary scratch (one host state at a time)
    DevBuf coo_off, coo_scratch, coo_groups, coo_terms, coo_nodes, coo_rows, coo_cols, coo_vals;
    uint64_t coo_uid = 0;  // observable whose groups/terms/offsets coo_* currently hold (0: none)
    std::map<std::pair<int, int>, qf_program*> basis_progs;  // (n, precision) -> per-qubit basis rotation program
    std::map<std::string, qf_program*> noise_progs;  // channel-free op runs of noise circuits (content key)
    int coo_n_groups = 0, coo_n_events = 0, coo_n_terms = 0;
    int64_t coo_total = 0;
    HostBuf pin;
    // NCCL
    NcclComm comm = nullptr;
    int rank = 0, world = 1;
    // stats (accumulated until qf_ctx_reset_stats); timing uses event pairs
    // recorded on the context stream and resolved lazily (no mid-call syncs)
    int timing = 0;  // 1: per kernel class, 2: + per launch (launch_ms)
    std::map<int, std::pair<double, long long>> launch_ms;  // launch id -> (ms, count)
    long long launches = 0;
    long long class_launches[4] = {0, 0, 0, 0};
    double ms[4] = {0, 0, 0, 0};
    double bytes[4] = {0, 0, 0, 0};
    double flops[4] = {0, 0, 0, 0};  // canonical algorithmic flops per class
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct PendingTime {
        size_t start, end;  // event pool indices
        int cls;            // class (< 4) or 100 + launch id
    };
    std::vector<PendingTime> pending;
    // CUDA graph of the last single-chunk evaluation, replayed while nothing it
    // captured (program, observable plan, buffers, batch) changes
    std::vector<const void*> graph_key;
    std::vector<const void*> graph_nocapture_key;  // configuration whose capture failed
    cudaGraphExec_t graph_exec = nullptr;
    long long graph_launches = 0;
};

namespace qfcapi {

int ensure_obs_dev(qf_observable* o, int prec, int kh, ObsDev& d, int t_begin, int t_end);
int check_thetas(const qf_program* prog, int batch, const double* thetas);
int stage_thetas(qf_ctx* ctx, const qf_program* prog, int batch, const double* thetas);
int forward_one(qf_ctx* ctx, qf_program* prog, const double* d_theta);  // forward pass of one row into ctx->psi

}  // namespace qfcapi
