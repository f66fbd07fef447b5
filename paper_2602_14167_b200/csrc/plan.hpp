// plan.hpp -- host-side compiler: circuit template -> fused tile sweeps,
// Pauli sum -> grouped term table.  Pure C++ (no CUDA) so it is unit-testable
// on the CPU through the C-ABI's introspection entry points.
#pragma once

#include <cstdint>
#include <string>
#include <functional>
#include <vector>

#include "plan.h"

namespace qfb {

struct GateSpec {  // one qf_op after validation
    int kind, q0, q1, slot;
    double coef, offset;
    int mat;
};

struct GateInfo {
    GateSpec g;
    int nw = 1;
    int wires[2] = {-1, -1};
    char wtype[2] = {'G', 'G'};  // per wire: 'D' diagonal, 'X', 'Y', 'G' general
    uint64_t need = 0;           // memory bits that must be register-resident
    bool diag = false;
    int gen = 0;                 // tap generator: 1 X, 2 Y, 3 Z, 4 ZZ, 0 none
};

struct PassPlan {
    int k = 0, R = 0;
    int n_taps = 0;
    std::vector<DevSweep> sweeps;
    std::vector<DevPhase> phases;
    std::vector<DevOp> ops;
    std::vector<DevTap> taps;  // global tap index -> (slot, coef)
    int max_mat = 0;           // max complex entries of any sweep matrix block
    int total_mat = 0;         // complex entries of all blocks (per-state matrix table)
    int max_ops = 0;           // max ops in a sweep
    int max_taps = 0;          // max taps in a sweep
};

struct ProgramPlan {
    int n = 0;
    int prec = 0;  // 0 = c64, 1 = c128
    int n_params = 0;
    std::vector<GateInfo> gates;
    std::vector<double> mats;  // constant matrices [n_mats][16][2]
    bool adjoint_ok = true;
    std::string adjoint_error;
    PassPlan fwd, bwd;
};

// Tile geometry per precision (64 KiB shared-memory tiles).
struct Geometry {
    int kf, Rf;   // forward tile bits / register bits
    int kb, Rb;   // adjoint (psi and lambda both resident)
    int kh;       // H|psi> tile bits
    int c;        // contiguous low bits (128-byte runs)
    int W;        // shared-memory swizzle width (bits)
};
Geometry geometry(int prec, int n);

// Returns "" on success, else the invalid-argument message.
std::string build_program_plan(int n, const std::vector<GateSpec>& ops, const double* mats,
                               int n_mats, int n_params, int prec, ProgramPlan& out);

struct ObservablePlan {
    int n = 0;
    int kh = 0;
    std::vector<DevGroup> groups;
    std::vector<DevTerm> terms;
    bool has_imag = false;
};
std::string build_observable_plan(int n, int n_terms, const int8_t* codes, const double* w_re,
                                  const double* w_im, int kh, ObservablePlan& out);

// Greedy list scheduler with a bit budget (exposed for tests/introspection).
// items: need masks; preds: predecessor lists (indices into items).
// Returns groups; each group = (bit mask used, ordered item list).
struct Group {
    uint64_t bits;
    std::vector<int> items;
};
std::vector<Group> schedule_groups(const std::vector<uint64_t>& need,
                                   const std::vector<std::vector<int>>& preds,
                                   uint64_t fixed_bits, int budget, int max_items = 0, bool search = false,
                                   int lookahead = 0, const std::function<double(const Group&)>* score = nullptr);

}  // namespace qfb
