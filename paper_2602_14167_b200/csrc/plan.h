// plan.h -- compiled execution plan shared by the host scheduler (plan.cpp) and
// the sm_100a kernels (kernels.cu).
//
// A circuit template (the reference's Circuit/GateInstruction list,
// include/qforge/circuit.hpp:14-83) is compiled ONCE into a sequence of fused
// tile sweeps.  A sweep streams every 2^k-amplitude tile of the state through
// shared memory exactly once and applies a run of gates whose non-diagonal
// bits all lie inside the tile.  Inside a sweep the tile is processed in
// phases: each thread holds 2^R amplitudes in registers spanning R "register
// bits" and applies every gate on those bits without touching shared memory;
// phases change the register bits with one swizzled shared-memory round trip.
// Diagonal gates (rz, rzz, z, s, cz) and cx controls never need a bit in
// registers: their bit values are known per amplitude.
//
// Bit positions are MEMORY positions: site q of an n-qubit register lives at
// bit n-1-q of the basis index (site 0 = most significant, circuit.cpp:87).
#pragma once

#ifndef __CUDACC_RTC__
#include <stdint.h>
#else
typedef unsigned char uint8_t;
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long size_t;
#endif

namespace qfb {

// Gate kinds: mirror of qf_gate (include/qforge_b200.h, = qforge::Gate,
// reference include/qforge/circuit.hpp:14-23); static_assert'ed in plan.cpp.
enum GateKind : int32_t {
    GK_H = 0, GK_X, GK_Y, GK_Z, GK_S, GK_RX, GK_RY, GK_RZ, GK_RZZ, GK_CX, GK_CZ,
    GK_SU4, GK_CSUM, GK_SUBSPACE_RY, GK_SUBSPACE_RZ, GK_UNITARY
};

constexpr int kMaxTileBits = 14;
constexpr int kMaxReg = 5;
constexpr int kMaxThreadBits = kMaxTileBits;

// Device op kinds (one entry per gate occurrence inside a phase).
enum DevKind : uint8_t {
    DK_G1 = 0,   // general 2x2 complex on register bit rb0
    DK_R1 = 1,   // real 2x2 (ry, h) on rb0
    DK_RX = 2,   // [[c, -i s], [-i s, c]] on rb0 (stored as c, s)
    DK_X1 = 3,   // Pauli X on rb0 (swap)
    DK_CX = 4,   // controlled X: target rb0, control pos0 (rb1 = its register bit or -1)
    DK_D1 = 5,   // diagonal on pos0 (rb0 = register bit or -1): d0, d1
    DK_D2 = 6,   // diagonal on pos0,pos1 (rb0/rb1 register bits or -1): d00 d01 d10 d11
    DK_G2 = 7,   // dense 4x4 on rb0 (wires[0], most significant local) and rb1
    // adjoint-gradient taps: accumulate Im<lambda|G|psi> into tap slot
    DK_TX = 8,   // G = X on rb0
    DK_TY = 9,   // G = Y on rb0
    DK_TZ = 10,  // G = Z on pos0 (rb0 register bit or -1)
    DK_TZZ = 11, // G = Z Z on pos0,pos1
    DK_RS = 12,  // real rotation [[c,-s],[s,c]] on rb0 applied as three shears; block (t, s), (sigma, 0):
                 // sigma = -1 means the kernel applies -R (a global phase)
    DK_NONE = 255
};

struct DevOp {
    uint8_t kind;
    int8_t rb0, rb1;   // register bit indices (0..R-1) or -1
    int8_t pos0, pos1; // memory bit positions or -1
    uint8_t pad;
    int16_t moff;      // offset (complex units) of this op's matrix in the sweep matrix block
    int32_t gate;      // program gate index (matrix source)
    int32_t tap;       // tap index local to the sweep, or -1
};

struct DevPhase {
    int32_t op_begin, op_end;
    int8_t reg_tl[kMaxReg];          // tile-local bit index of register bit r
    int8_t thr_tl[kMaxThreadBits];   // tile-local bit index of thread-id bit t
    int8_t pad[3];
};

struct DevSweep {
    int32_t k;             // tile bits
    int32_t R;             // register bits
    int32_t n_phases;
    int32_t phase_begin;
    int32_t op_begin, op_end;   // all ops of the sweep (matrix prologue)
    int32_t n_mat;              // complex entries of the sweep matrix block
    int32_t mbase;              // offset of the block in the pass's per-state matrix table
    int32_t tap_begin, n_taps;  // taps of this sweep (global numbering)
    uint32_t out_mask;          // memory bits not in the tile
    int8_t tb[kMaxTileBits];    // tile-local bit -> memory bit position
    int8_t pad[2];
};

// Gate table entry (device copy of the program's gates).
struct DevGate {
    int32_t kind;      // qf_gate numbering
    int32_t slot;      // theta slot or -1
    double coef, offset;
    int32_t mat;       // constant matrix index or -1
    int32_t q0, q1;
};

// Tap -> parameter mapping for the gradient reduction: grad[slot] += coef * tap.
struct DevTap {
    int32_t slot;
    int32_t pad;
    double coef;
};

// ---- H|psi> ----
// Terms are grouped by the flip bits above the tile (f_out); each group reads
// one partner tile (tile_index ^ (f_out >> k)).
enum TermKind : int32_t { TK_DIAG = 0, TK_FLIP = 1, TK_GEN = 2 };

struct DevTerm {
    int32_t kind;
    uint32_t f_in;     // flip bits inside the tile
    uint32_t z;        // z mask (all bits)
    uint32_t fz_par;   // parity(f & z) & 1 (folded into the sign)
    int32_t yodd;      // odd number of Y: the coefficient is purely imaginary
    double c_re, c_im; // Re(w) * i^y  (Hermitian part)
    double ci_re, ci_im; // Im(w) * i^y (imaginary part of expectation_pauli)
};

struct DevGroup {
    uint32_t f_out;    // flip bits above the tile
    int32_t term_begin, term_end;
    int32_t pad;
};

// Kernel arguments of one H|psi> launch (AOT kernel and NVRTC kernels).
struct HArgs {
    const void* psi;
    void* lam;
    int n, kh;
    const DevGroup* groups;
    int n_groups;
    const DevTerm* terms;
    int write_lam;
    int use_imag;
    double* epart;             // [B][tiles]
    int prefetch;              // generic kernel: double-buffer partner tiles (few terms per group)
    int tma;                   // generic kernel, with prefetch: partner tiles by TMA bulk copy + mbarrier
};

// Kernel arguments of one sweep launch (AOT interpreter and NVRTC kernels).
struct SweepArgs {
    void* psi;                 // [B][N] complex (float2 / double2)
    void* lam;                 // adjoint state (backward only)
    const double* theta;       // [B_total][P]
    int P;
    int n;
    int batch_offset;          // global index of blockIdx.y == 0 (theta rows)
    int from_zero;             // forward sweep 0 builds |0..0> in-tile
    DevSweep sw;               // this sweep (by value)
    const DevPhase* phases;
    const DevOp* ops;
    const DevGate* gates;
    const double* cmats;       // constant matrices [n][16][2]
    double* tap_part;          // [B][n_taps_total][tiles]
    int n_taps_total;
    const void* gmat;          // per-state gate-matrix table [B][gmat_stride] complex (RT)
    int gmat_stride;           // complex entries per state (forward block then adjoint block)
    int gmat_pass_base;        // offset of this pass's block inside a state's table
    int batch;                 // states in this launch (persistent kernels)
};

}  // namespace qfb
