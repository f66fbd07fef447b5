// jit.hpp -- per-program specialised sweep kernels (NVRTC, sm_100a).
//
// The AOT interpreter (sweep_impl.cuh) dispatches every gate at run time; the
// specialised kernels bake the whole sweep (tile bits, phases, gate order,
// register bits) into straight-line code: no dispatch, no register moves for
// permutation gates, full cross-gate instruction-level parallelism.  Kernels are
// generated from the plan, compiled with NVRTC on worker threads, cached on disk
// by source hash, and loaded with cudaLibraryLoadData.
#pragma once

#include <string>
#include <vector>

#include "plan.hpp"

namespace qfb {

struct JitKernel {
    void* kernel = nullptr;  // cudaKernel_t
    int threads = 0;
    size_t smem = 0;
    bool pipe = false;       // persistent, cp.async double-buffered variant
    int ctas = 0;            // resident CTAs (pipe mode grid)
    std::string module;      // key of the loaded module in the process-wide table ("" = none)
};

// Loaded modules are shared process-wide by source hash (identical kernels of
// different programs load once) and reference-counted: every JitKernel that
// holds one is released exactly once (program / observable destruction, plan
// rebuild), and the module is unloaded with its last user.
void jit_release(JitKernel& k);
void jit_release(std::vector<JitKernel>& ks);

bool jit_pipe_mode(const PassPlan& pass, int si);

struct JitPass {
    std::vector<JitKernel> sweeps;
    bool ok = false;
};

struct JitStats {
    double seconds = 0.0;
    int compiled = 0, cached = 0;
    std::string error;
};

// Source of the specialised kernel for sweep `si` of `pass` (exposed for tests).
std::string jit_source(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd);
size_t jit_smem_bytes(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd);
int jit_tap_stage(const ProgramPlan& P, const PassPlan& pass, int si, bool bwd);

// NVRTC compile of one generated source to an sm_100a cubin (no GPU needed).
bool jit_compile_source(const std::string& src, std::string& cubin, std::string& err);

// Builds (or loads from the cache) every sweep kernel of both passes.
// Returns false and fills st.error if NVRTC is unavailable or a compile fails.
// load_modules = false: compile into the disk cache only (no device needed)
bool jit_build(const ProgramPlan& P, JitPass& fwd, JitPass& bwd, JitStats& st, bool load_modules = true);

// Launch one specialised sweep.
int jit_launch(const JitKernel& k, const SweepArgs& a, int tiles, int batch, void* stream);
const std::string& jit_last_launch_detail();  // configuration of the last failed jit_launch

// Specialised H|psi> + energy kernel of one observable (qf_hpsi); at most
// kJitHpsiMaxTerms terms (larger sums keep the AOT hpsi_kernel).
constexpr int kJitHpsiMaxTerms = 256;
std::string jit_hpsi_source(const ObservablePlan& O, int prec);
bool jit_build_hpsi(const ObservablePlan& O, int prec, JitKernel& out, std::string& err);
int jit_launch_hpsi(const JitKernel& k, const HArgs& a, int tiles, int batch, void* stream);

}  // namespace qfb
