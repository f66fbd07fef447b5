// plan.cpp -- circuit template -> fused tile sweeps (see plan.h for the model).
//
// Replaces the reference's per-energy-call rebuild of the op list
// (variational.cpp:41 -> builder -> Circuit::gate, circuit.cpp:178-186) and the
// one-sweep-per-gate loop of run() (circuit.cpp:313-315): the template is
// validated and scheduled once, then executed for every parameter set.
#include "plan.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <complex>
#include <functional>
#include <map>
#include <set>

#include "../../include/qforge_b200.h"

namespace qfb {

static_assert((int)GK_H == (int)QF_H && (int)GK_RX == (int)QF_RX && (int)GK_RZZ == (int)QF_RZZ && (int)GK_CX == (int)QF_CX &&
                  (int)GK_SU4 == (int)QF_SU4 && (int)GK_UNITARY == (int)QF_UNITARY,
              "GateKind must mirror qf_gate");

Geometry geometry(int prec, int n) {
    Geometry g;
    if (prec == QF_C128) {
        g.kf = 12; g.Rf = 4; g.kb = 11; g.Rb = 3; g.kh = 11; g.c = 3; g.W = 3;
    } else {
        g.kf = 13; g.Rf = 5; g.kb = 12; g.Rb = 4; g.kh = 12; g.c = 4; g.W = 4;
    }
    // development override: QF_GEOM_C64 / QF_GEOM_C128 = "kf,Rf,kb,Rb"
    bool overridden = false;
    if (const char* e = std::getenv(prec == QF_C128 ? "QF_GEOM_C128" : "QF_GEOM_C64")) {
        int a, b, c, d;
        if (std::sscanf(e, "%d,%d,%d,%d", &a, &b, &c, &d) == 4) {
            g.kf = a; g.Rf = b; g.kb = c; g.Rb = d;
            overridden = true;
        }
    }
    g.kf = std::min(g.kf, n);
    g.kb = std::min(g.kb, n);
    // Small states (one tile, or a few, per state): a tile's 2^(k - R) threads are
    // all the parallelism a state gets, so keep >= 256 threads per tile by trading
    // register bits for threads (more phases, each cheaper).  C1 (n = 10, batch
    // 16): 271 k -> 533 k evals/s (tools/r2_c1g.sh).
    if (!overridden && n <= 12) {
        g.Rf = std::max(2, std::min(g.Rf, g.kf - 8));
        g.Rb = std::max(2, std::min(g.Rb, g.kb - 8));
    }
    g.kh = std::min(g.kh, n);
    g.Rf = std::min(g.Rf, g.kf);
    g.Rb = std::min(g.Rb, g.kb);
    g.c = std::min(g.c, n);
    g.c = std::max(0, std::min(g.c, std::min(g.kf, g.kb) - 2));  // leave room for 2-qubit gates
    return g;
}

static int popc(uint64_t x) { return __builtin_popcountll(x); }

// development A/B toggles: VAR=0 turns the feature off
static bool env_flag_off(const char* name) {
    const char* e = std::getenv(name);
    return e && e[0] == '0';
}

// Incremental form of the group scheduler (sweeps are chosen one at a time so the
// caller can hand a sweep's light tail phase back before the next one is chosen).
class GroupScheduler {
public:
    GroupScheduler(const std::vector<uint64_t>& need, const std::vector<std::vector<int>>& preds, uint64_t fixed_bits,
                   int budget, int max_items, bool search, int lookahead,
                   const std::function<double(const Group&)>* score)
        : need_(need), fixed_(fixed_bits), budget_(budget), max_items_(max_items), search_(search),
          lookahead_(lookahead), score_(score) {
        const int n = (int)need.size();
        succ_.resize(n);
        st_.indeg.assign(n, 0);
        for (int j = 0; j < n; ++j) {
            st_.indeg[j] = (int)preds[j].size();
            for (int p : preds[j]) succ_[p].push_back(j);
        }
        for (int j = 0; j < n; ++j)
            if (st_.indeg[j] == 0) st_.ready.insert(j);
        st_.remaining = n;
        uint64_t all_bits = fixed_bits;
        for (uint64_t m : need) all_bits |= m;
        nb_ = all_bits ? 64 - __builtin_clzll(all_bits) : 0;
        win_ = budget - popc(fixed_bits);
    }
    int remaining() const { return st_.remaining; }
    // Give items of the last group back (they were taken last; none of their
    // successors was taken).
    void untake(const std::vector<int>& items) {
        std::set<int> back(items.begin(), items.end());
        for (int u : items) {
            ++st_.remaining;
            for (int sc : succ_[u]) {
                if (st_.indeg[sc] == 0) st_.ready.erase(sc);
                ++st_.indeg[sc];
            }
        }
        for (int u : items)
            if (st_.indeg[u] == 0) st_.ready.insert(u);
    }
    // Choose and take the next group; false when nothing fits the budget.
    bool next(Group& out) {
        State s_best = st_;
        Group g = greedy(s_best);
        if (search_ && win_ > 0) choose(g, s_best);
        if (g.items.empty()) return false;  // an item needs more bits than the budget
        st_ = std::move(s_best);
        out = std::move(g);
        return true;
    }

private:
    struct State {
        std::set<int> ready;
        std::vector<int> indeg;
        int remaining = 0;
    };
    void take(State& S, Group& g, int it) const {
        S.ready.erase(it);
        g.items.push_back(it);
        --S.remaining;
        for (int sc : succ_[it])
            if (--S.indeg[sc] == 0) S.ready.insert(sc);
    }
    // greedy: absorb every ready item that fits, then widen the group's bits by the
    // ready item that needs the fewest extra bits, until the budget is spent
    Group greedy(State& S) const {
        Group g;
        g.bits = fixed_;
        for (;;) {
            bool progress = true;
            while (progress && (max_items_ <= 0 || (int)g.items.size() < max_items_)) {
                progress = false;
                for (int it : S.ready) {
                    if ((need_[it] & ~g.bits) == 0) {
                        take(S, g, it);
                        progress = true;
                        break;
                    }
                }
            }
            int best = -1, best_cost = 1 << 30;
            if (max_items_ > 0 && (int)g.items.size() >= max_items_) break;
            for (int it : S.ready) {
                int extra = popc(need_[it] & ~g.bits);
                if (popc(g.bits) + extra <= budget_ && extra < best_cost) {
                    best = it;
                    best_cost = extra;
                }
            }
            if (best < 0) break;
            g.bits |= need_[best];
        }
        return g;
    }
    // closure of fixed bits: every item reachable through items that fit
    Group absorb(State& S, uint64_t bits) const {
        Group g;
        g.bits = bits;
        bool progress = true;
        while (progress) {
            progress = false;
            for (auto itr = S.ready.begin(); itr != S.ready.end();) {
                if (max_items_ > 0 && (int)g.items.size() >= max_items_) return g;
                const int it = *itr;
                if ((need_[it] & ~bits) == 0) {
                    take(S, g, it);
                    progress = true;
                    itr = S.ready.lower_bound(it);
                } else {
                    ++itr;
                }
            }
        }
        return g;
    }
    void choose(Group& g, State& s_best) const {
        // candidate bit sets: every win-subset of the free bits when there are few
        // (C(13, 5) = 1287 at most for phases), else windows of consecutive bits
        std::vector<uint64_t> cands;
        const uint64_t freeb = (nb_ >= 64 ? ~0ull : ((1ull << nb_) - 1)) & ~fixed_;
        static const bool exhaustive = !(std::getenv("QF_PHASE_SEARCH") && std::getenv("QF_PHASE_SEARCH")[0] == 'w');
        if (exhaustive && popc(freeb) <= 14) {
            std::vector<int> fb;
            for (int b = 0; b < nb_; ++b)
                if (freeb >> b & 1) fb.push_back(b);
            const int m = (int)fb.size();
            for (uint32_t sel = 0; sel < (1u << m); ++sel) {
                if (__builtin_popcount(sel) != win_) continue;
                uint64_t wbits = 0;
                for (int i = 0; i < m; ++i)
                    if (sel >> i & 1) wbits |= 1ull << fb[i];
                cands.push_back(wbits);
            }
        } else {
            for (int s0 = 0; s0 + win_ <= nb_; ++s0) {
                const uint64_t wbits = (((win_ >= 64) ? ~0ull : ((1ull << win_) - 1)) << s0);
                if (!(wbits & fixed_)) cands.push_back(wbits);
            }
        }
        std::vector<std::pair<int, uint64_t>> scored;  // (closure size, bits)
        for (uint64_t wb : cands) {
            State s2 = st_;
            scored.push_back({(int)absorb(s2, fixed_ | wb).items.size(), wb});
        }
        if (lookahead_ > 0 && !scored.empty()) {
            // two-level: among the best `lookahead` first choices, the one whose
            // closure plus the best next closure covers the most items
            std::stable_sort(scored.begin(), scored.end(),
                             [](const auto& x, const auto& y) { return x.first > y.first; });
            int best_total = -1;
            for (size_t c = 0; c < scored.size() && (int)c < lookahead_; ++c) {
                State s2 = st_;
                Group g1 = absorb(s2, fixed_ | scored[c].second);
                int second = 0;
                if (s2.remaining > 0)
                    for (uint64_t wb : cands) {
                        State s3 = s2;
                        second = std::max(second, (int)absorb(s3, fixed_ | wb).items.size());
                    }
                const int total = (int)g1.items.size() + second;
                if (total > best_total && g1.items.size() >= g.items.size()) {
                    best_total = total;
                    g = std::move(g1);
                    s_best = std::move(s2);
                }
            }
        } else if (score_) {
            // caller's cost model (e.g. gates per phase of the resulting sweep)
            double best = (*score_)(g);
            for (auto& sc : scored) {
                State s2 = st_;
                Group gw = absorb(s2, fixed_ | sc.second);
                const double v = (*score_)(gw);
                if (v > best) {
                    best = v;
                    g = std::move(gw);
                    s_best = std::move(s2);
                }
            }
        } else {
            for (auto& sc : scored)
                if (sc.first > (int)g.items.size()) {
                    State s2 = st_;
                    g = absorb(s2, fixed_ | sc.second);
                    s_best = std::move(s2);
                }
        }
    }

    const std::vector<uint64_t>& need_;
    std::vector<std::vector<int>> succ_;
    State st_;
    uint64_t fixed_;
    int budget_, max_items_;
    bool search_;
    int lookahead_;
    const std::function<double(const Group&)>* score_;
    int nb_ = 0, win_ = 0;
};

std::vector<Group> schedule_groups(const std::vector<uint64_t>& need,
                                   const std::vector<std::vector<int>>& preds,
                                   uint64_t fixed_bits, int budget, int max_items, bool search, int lookahead,
                                   const std::function<double(const Group&)>* score) {
    GroupScheduler gs(need, preds, fixed_bits, budget, max_items, search, lookahead, score);
    std::vector<Group> out;
    while (gs.remaining() > 0) {
        Group g;
        if (!gs.next(g)) return {};
        out.push_back(std::move(g));
    }
    return out;
}

static bool commute(const GateInfo& a, const GateInfo& b) {
    for (int i = 0; i < a.nw; ++i)
        for (int j = 0; j < b.nw; ++j)
            if (a.wires[i] == b.wires[j]) {
                char ta = a.wtype[i], tb = b.wtype[j];
                if (ta != tb || ta == 'G') return false;
            }
    return true;
}

static bool is_diag_matrix(const double* m, int d) {  // exact-zero test, circuit.cpp:90-95
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c)
            if (r != c && (m[2 * (r * 4 + c)] != 0.0 || m[2 * (r * 4 + c) + 1] != 0.0)) return false;
    return true;
}

static bool is_unitary(const double* m, int d) {  // Circuit::unitary check, circuit.cpp:193-196
    using cd = std::complex<double>;
    double worst = 0.0;
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            cd acc = 0.0;
            for (int k = 0; k < d; ++k)
                acc += std::conj(cd(m[2 * (k * 4 + r)], m[2 * (k * 4 + r) + 1])) *
                       cd(m[2 * (k * 4 + c)], m[2 * (k * 4 + c) + 1]);
            worst = std::max(worst, std::abs(acc - cd(r == c ? 1.0 : 0.0, 0.0)));
        }
    return worst < 1e-10;
}

static std::string classify(int n, const GateSpec& s, const double* mats, int n_mats,
                            int n_params, GateInfo& gi) {
    gi.g = s;
    auto inr = [n](int q) { return q >= 0 && q < n; };
    const bool two = s.kind == QF_RZZ || s.kind == QF_CX || s.kind == QF_CZ ||
                     s.kind == QF_SU4 || (s.kind == QF_UNITARY && s.q1 >= 0);
    switch (s.kind) {
        case QF_H: case QF_X: case QF_Y: case QF_Z: case QF_S:
        case QF_RX: case QF_RY: case QF_RZ: case QF_RZZ:
        case QF_CX: case QF_CZ: case QF_SU4: case QF_UNITARY:
            break;
        case QF_CSUM: case QF_SUBSPACE_RY: case QF_SUBSPACE_RZ:
            return "gate_matrix: qudit gates are not supported on the qubit device path";
        default:
            return "gate_matrix: unknown gate kind";
    }
    if (!inr(s.q0)) return "Circuit: wire out of range";
    if (two) {
        if (!inr(s.q1)) return "Circuit: wire out of range";
        if (s.q0 == s.q1) return "Circuit: duplicate wires";
    }
    gi.nw = two ? 2 : 1;
    gi.wires[0] = s.q0;
    gi.wires[1] = two ? s.q1 : -1;
    if (s.slot >= n_params) return "program: parameter slot out of range";
    if (s.slot < 0 && !std::isfinite(s.offset)) return "Circuit: non-finite parameter";
    if (s.slot >= 0 && (!std::isfinite(s.coef) || !std::isfinite(s.offset)))
        return "Circuit: non-finite parameter";
    if (s.kind == QF_SU4 || s.kind == QF_UNITARY) {
        if (s.slot >= 0)
            return "program: parameterised su4/unitary gates are not supported on the device path";
        if (s.mat < 0 || s.mat >= n_mats || !mats) return "program: missing gate matrix";
        const double* m = mats + 32 * (size_t)s.mat;
        if (!is_unitary(m, two ? 4 : 2)) return "unitary: matrix is not unitary";
        gi.diag = is_diag_matrix(m, two ? 4 : 2);
    }
    auto pos = [n](int q) { return n - 1 - q; };
    switch (s.kind) {
        case QF_Z: case QF_S: case QF_RZ: case QF_RZZ: case QF_CZ:
            gi.diag = true;
            break;
        default:
            break;
    }
    if (gi.diag) {
        gi.wtype[0] = gi.wtype[1] = 'D';
        gi.need = 0;
    } else if (s.kind == QF_X || s.kind == QF_RX) {
        gi.wtype[0] = 'X';
        gi.need = 1ull << pos(s.q0);
    } else if (s.kind == QF_Y || s.kind == QF_RY) {
        gi.wtype[0] = 'Y';
        gi.need = 1ull << pos(s.q0);
    } else if (s.kind == QF_CX) {
        gi.wtype[0] = 'D';
        gi.wtype[1] = 'X';
        gi.need = 1ull << pos(s.q1);
    } else {
        gi.wtype[0] = gi.wtype[1] = 'G';
        gi.need = 1ull << pos(s.q0);
        if (two) gi.need |= 1ull << pos(s.q1);
    }
    if (s.slot >= 0) {
        switch (s.kind) {
            case QF_RX: gi.gen = 1; break;
            case QF_RY: gi.gen = 2; break;
            case QF_RZ: gi.gen = 3; break;
            case QF_RZZ: gi.gen = 4; break;
            default: gi.gen = 0; break;  // slot feeds a parameter-free gate: zero derivative
        }
    }
    return "";
}

static int mat_size(uint8_t kind) {
    switch (kind) {
        case DK_G1: case DK_R1: case DK_RX: return 4;
        case DK_RS: return 2;
        case DK_D1: return 2;
        case DK_D2: return 4;
        case DK_G2: return 16;
        default: return 0;
    }
}

// Warp-index bits of every phase of a sweep (tile-local bit mask; 0 = no choice).
// Greedy runs: a run of phases keeps one set of nwb warp bits, taken from the
// tile bits none of the run's phases needs in registers (and never the `low`
// lowest tile bits, which must stay lanes for the direct HBM phases).  Within a
// run's candidates the set whose leftover lane bits cover the most distinct
// residues mod W (shared-memory bank spread) wins, then the highest bits.
// QF_WARP_RUNS=0 turns it off (development A/B).
static std::vector<uint64_t> warp_bit_runs(const std::vector<Group>& phases, int k, int R, int W, int low) {
    std::vector<uint64_t> out(phases.size(), 0);
    const int nwb = (k - R) - 5;
    static const bool off = std::getenv("QF_WARP_RUNS") && std::getenv("QF_WARP_RUNS")[0] == '0';
    if (off || nwb <= 0 || phases.size() < 2) return out;
    const uint64_t tile = (1ull << k) - 1, lowm = (1ull << low) - 1;
    size_t f = 0;
    while (f < phases.size()) {
        uint64_t allowed = tile & ~phases[f].bits & ~lowm;
        size_t g = f;
        while (g + 1 < phases.size() && popc(allowed & ~phases[g + 1].bits) >= nwb) allowed &= ~phases[++g].bits;
        if (popc(allowed) < nwb) {  // cannot happen for k - R - low >= nwb; keep the default assignment
            f = g + 1;
            continue;
        }
        std::vector<int> cand;
        for (int b = 0; b < k; ++b)
            if (allowed >> b & 1) cand.push_back(b);
        uint64_t best = 0;
        long best_score = -1;
        const size_t m = cand.size();
        for (uint64_t sel = 0; sel < (1ull << m); ++sel) {  // m <= k - R - low (small)
            if (popc(sel) != nwb) continue;
            uint64_t w = 0;
            for (size_t i = 0; i < m; ++i)
                if (sel >> i & 1) w |= 1ull << cand[i];
            long score = 0;
            for (size_t h = f; h <= g; ++h) {
                // this phase's lanes: the free bits left after registers (padded high) and warps
                uint64_t r = phases[h].bits;
                for (int b = k - 1; b >= 0 && popc(r) < R; --b)
                    if (!(w >> b & 1)) r |= 1ull << b;
                const uint64_t lanes = tile & ~r & ~w;
                uint32_t res = 0;
                for (int b = 0; b < k; ++b)
                    if (lanes >> b & 1) res |= 1u << (b % W);
                score += popc(res);
            }
            score = score * 4096 + (long)(w >> 1);  // tie-break: higher bits
            if (score > best_score) {
                best_score = score;
                best = w;
            }
        }
        for (size_t h = f; h <= g; ++h) out[h] = best;
        f = g + 1;
    }
    return out;
}

// Lower one pass (forward or adjoint) of an ordered gate list.
static void lower_pass(const ProgramPlan& P, const std::vector<int>& order,
                       const std::vector<std::vector<int>>& preds_in_order, int k, int R,
                       int c, int W, bool adjoint, PassPlan& out) {
    const int n = P.n;
    out.k = k;
    out.R = R;
    std::vector<uint64_t> need(order.size());
    for (size_t i = 0; i < order.size(); ++i) need[i] = P.gates[order[i]].need;
    const uint64_t all = (n >= 64) ? ~0ull : ((1ull << n) - 1);
    const uint64_t fixed = (n <= k) ? all : ((1ull << c) - 1);
    // cap the gates per sweep: the specialised kernels are straight-line code, and
    // very long sweeps overflow the instruction cache
    // Cap on gates per sweep.  The generated kernels are straight-line code and
    // ptxas time grows faster than linearly with their length.  With the tile and
    // phase searches, 200 ops costs nothing at run time against no cap (C2 181.6
    // vs 181.1 ms per step) and bounds pathological sweeps; 120 would halve C2's
    // cold NVRTC build (21.0 -> 8.5 s on the GPU host) for 2.5 % C2 / 1.7 % C5
    // throughput (tools/r2_p11.sh).  QF_MAX_SWEEP_OPS=n overrides (0 = no cap).
    int max_ops = 200;
    if (const char* e = std::getenv("QF_MAX_SWEEP_OPS")) max_ops = std::atoi(e);
    // Sweep tiles: besides the greedy tile, every window of consecutive memory
    // bits above the fixed ones; the tile whose closure holds the most gates wins.
    // For the layered ansatz this follows the light-cone staircase (C2: 6 + 7
    // sweeps instead of 10 + 14 under the 120-op cap).  Together with the phase
    // search it pays: C2 194.7 -> 184.5 ms per step, C3 +11 %, C5 +3 %; alone
    // (greedy phases) it did not (profiles/r2_sweep_experiments.md).
    // QF_SWEEP_SEARCH=0: greedy only; QF_SWEEP_LOOKAHEAD=K: two-level choice.
    static const bool sweep_search = !(std::getenv("QF_SWEEP_SEARCH") && std::getenv("QF_SWEEP_SEARCH")[0] == '0');
    static const int sweep_look = [] {
        const char* e = std::getenv("QF_SWEEP_LOOKAHEAD");
        return e ? std::atoi(e) : 0;
    }();
    // QF_SWEEP_OBJ=ratio: score a candidate tile by gates per phase of the sweep it
    // would make (its closure scheduled into phases), cost floored at 1.5 phases
    // for the HBM pass (development A/B)
    static const char* obj_env = std::getenv("QF_SWEEP_OBJ");
    const bool ratio_obj = obj_env && (std::string(obj_env) == "ratio" || (std::string(obj_env) == "ratio_fwd" && !adjoint));
    std::function<double(const Group&)> ratio_score = [&](const Group& gw) -> double {
        if (gw.items.empty()) return -1.0;
        uint64_t bits = gw.bits;
        for (int p = 0; p < n && popc(bits) < k; ++p) bits |= 1ull << p;
        int tl[64];
        int t = 0;
        for (int p = 0; p < 64; ++p) tl[p] = (bits >> p & 1) ? t++ : -1;
        std::map<int, int> loc;
        for (size_t i = 0; i < gw.items.size(); ++i) loc[gw.items[i]] = (int)i;
        std::vector<uint64_t> ln(gw.items.size());
        std::vector<std::vector<int>> lp(gw.items.size());
        for (size_t i = 0; i < gw.items.size(); ++i) {
            const int it = gw.items[i];
            for (int p = 0; p < n; ++p)
                if (need[it] >> p & 1) ln[i] |= 1ull << tl[p];
            for (int pr : preds_in_order[it]) {
                auto f = loc.find(pr);
                if (f != loc.end()) lp[i].push_back(f->second);
            }
        }
        const auto ph = schedule_groups(ln, lp, 0, R, 0, true);
        return (double)gw.items.size() / std::max(1.5, (double)ph.size());
    };
    GroupScheduler gsched(need, preds_in_order, fixed, k, max_ops, sweep_search, sweep_look,
                          ratio_obj ? &ratio_score : nullptr);
    // A sweep whose last phase is a light tail (at most `tail_max` gates that need
    // register bits) hands that phase's gates back to the next sweep, saving a
    // shared-memory exchange (QF_TAIL_MAX, development A/B; -1 = off).
    static const int tail_max = [] {
        const char* e = std::getenv("QF_TAIL_MAX");
        return e ? std::atoi(e) : -1;
    }();
    Group sw;
    while (gsched.remaining() > 0) {
        if (!gsched.next(sw)) {
            out.sweeps.clear();  // an item needs more bits than the tile (reported by the caller)
            return;
        }
        // pad the tile to exactly k bits with the lowest free positions
        uint64_t bits = sw.bits;
        for (int p = 0; p < n && popc(bits) < k; ++p) bits |= 1ull << p;
        DevSweep ds{};
        ds.k = k;
        ds.R = R;
        int tl_of_pos[64];
        for (int p = 0; p < 64; ++p) tl_of_pos[p] = -1;
        int t = 0;
        for (int p = 0; p < n; ++p)
            if (bits >> p & 1) {
                ds.tb[t] = (int8_t)p;
                tl_of_pos[p] = t++;
            }
        ds.out_mask = (uint32_t)(all & ~bits);
        ds.phase_begin = (int)out.phases.size();
        ds.op_begin = (int)out.ops.size();
        ds.tap_begin = out.n_taps;

        // phases: schedule the sweep's gates over tile-local bits with budget R
        auto order_of = [&](int it) { return order[it]; };
        std::map<int, int> local;  // index in `order` -> index in sweep
        for (size_t i = 0; i < sw.items.size(); ++i) local[sw.items[i]] = (int)i;
        std::vector<uint64_t> lneed(sw.items.size());
        std::vector<std::vector<int>> lpreds(sw.items.size());
        for (size_t i = 0; i < sw.items.size(); ++i) {
            int it = sw.items[i];
            uint64_t m = 0;
            for (int p = 0; p < n; ++p)
                if (need[it] >> p & 1) m |= 1ull << tl_of_pos[p];
            lneed[i] = m;
            for (int pr : preds_in_order[it]) {
                auto f = local.find(pr);
                if (f != local.end()) lpreds[i].push_back(f->second);
            }
        }
        // phases: each one takes the register-bit set whose closure holds the most
        // gates (every R-subset of the tile bits; the greedy choice wins ties):
        // fewer phases means fewer shared-memory exchanges, C2 36 + 39 -> 30 + 36
        // phases and 205.2 -> 198.0 ms per step.  QF_PHASE_SEARCH=0: greedy only,
        // =w: windows of consecutive tile bits only (development A/B).
        static const bool phase_search = !(std::getenv("QF_PHASE_SEARCH") && std::getenv("QF_PHASE_SEARCH")[0] == '0');
        static const int phase_look = [] {
            const char* e = std::getenv("QF_PHASE_LOOKAHEAD");
            return e ? std::atoi(e) : 0;
        }();
        auto phases = schedule_groups(lneed, lpreds, 0, R, 0, phase_search, phase_look);
        if (tail_max >= 0 && phases.size() > 1) {
            int nd = 0;
            for (int li : phases.back().items) nd += lneed[li] != 0;
            if (nd <= tail_max) {
                std::vector<int> back;
                for (int li : phases.back().items) back.push_back(sw.items[li]);
                gsched.untake(back);
                phases.pop_back();
            }
        }
        // Inside a phase, issue ready non-diagonal gates first and release the
        // diagonal ones (which commute with each other) in batches: long runs of
        // diagonal gates and Z taps are fused by the kernel generator.
        for (auto& ph : phases) {
            std::map<int, int> pos;  // local item -> position in phase
            for (size_t i = 0; i < ph.items.size(); ++i) pos[ph.items[i]] = (int)i;
            std::vector<int> indeg(ph.items.size(), 0);
            std::vector<std::vector<int>> succ(ph.items.size());
            for (size_t i = 0; i < ph.items.size(); ++i)
                for (int pr : lpreds[ph.items[i]]) {
                    auto f = pos.find(pr);
                    if (f == pos.end()) continue;
                    ++indeg[i];
                    succ[f->second].push_back((int)i);
                }
            std::set<int> ready;
            for (size_t i = 0; i < ph.items.size(); ++i)
                if (!indeg[i]) ready.insert((int)i);
            std::vector<int> order;
            auto take = [&](int i) {
                ready.erase(i);
                order.push_back(ph.items[i]);
                for (int s2 : succ[i])
                    if (--indeg[s2] == 0) ready.insert(s2);
            };
            while (!ready.empty()) {
                int pick = -1;
                for (int i : ready)
                    if (!P.gates[order_of(sw.items[ph.items[i]])].diag) { pick = i; break; }
                if (pick >= 0) {
                    take(pick);
                    continue;
                }
                std::vector<int> diag(ready.begin(), ready.end());  // all ready are diagonal
                for (int i : diag) take(i);
            }
            ph.items.swap(order);
        }
        // Warp-index thread bits (above the 5 lane bits) are held on the same tile
        // bits over runs of phases: a phase change that keeps them permutes data
        // only inside each warp's own region of the shared tile, so the generated
        // kernel syncs that warp (__syncwarp) instead of the whole CTA there.
        const std::vector<uint64_t> wbits = warp_bit_runs(phases, k, R, W, P.prec == QF_C128 ? 1 : 2);
        int moff = 0, ntap = 0;
        for (size_t fi = 0; fi < phases.size(); ++fi) {
            auto& ph = phases[fi];
            const uint64_t wb = wbits[fi];
            DevPhase dp{};
            for (int i = 0; i < kMaxReg; ++i) dp.reg_tl[i] = -1;
            for (int i = 0; i < kMaxThreadBits; ++i) dp.thr_tl[i] = -1;
            // register bits: the needed ones, padded with the highest free tile bits
            uint64_t rbits = ph.bits;
            for (int b = k - 1; b >= 0 && popc(rbits) < R; --b)
                if (!(wb >> b & 1)) rbits |= 1ull << b;
            int r = 0;
            int rb_of_tl[kMaxTileBits];
            for (int b = 0; b < kMaxTileBits; ++b) rb_of_tl[b] = -1;
            for (int b = 0; b < k; ++b)
                if (rbits >> b & 1) {
                    dp.reg_tl[r] = (int8_t)b;
                    rb_of_tl[b] = r++;
                }
            // thread bits: lanes first, covering distinct residues mod W (bank spread)
            std::vector<int> free_bits;
            for (int b = 0; b < k; ++b)
                if (!(rbits >> b & 1) && !(wb >> b & 1)) free_bits.push_back(b);
            std::vector<int> lanes, rest;
            std::vector<bool> used(free_bits.size(), false);
            const int nl = std::min<int>(5, (int)free_bits.size());
            for (int pass = 0; pass < 2 && (int)lanes.size() < nl; ++pass) {
                uint32_t seen = 0;
                for (int l : lanes) seen |= 1u << (l % W);
                for (size_t i = 0; i < free_bits.size() && (int)lanes.size() < nl; ++i) {
                    if (used[i]) continue;
                    int res = free_bits[i] % W;
                    if (pass == 0 && (seen >> res & 1)) continue;
                    used[i] = true;
                    seen |= 1u << res;
                    lanes.push_back(free_bits[i]);
                }
            }
            for (size_t i = 0; i < free_bits.size(); ++i)
                if (!used[i]) rest.push_back(free_bits[i]);
            std::sort(lanes.begin(), lanes.end());
            // One shared-memory wavefront serves 2^W consecutive lanes (128 B of 8- or
            // 16-byte amplitudes), so the first W lane slots must land in distinct bank
            // groups: under the XOR-fold swizzle tile bit b moves bank group b mod W.
            // Distinct residues go first; a repeated residue takes a higher lane bit,
            // where it only selects the wavefront.  (Global coalescing does not care
            // about lane order: the warp still covers the same sectors.)
            if (!env_flag_off("QF_LANE_ORDER")) {
                std::vector<int> first, later;
                uint32_t seen = 0;
                for (int l : lanes) {
                    if ((int)first.size() < W && !(seen >> (l % W) & 1)) {
                        seen |= 1u << (l % W);
                        first.push_back(l);
                    } else {
                        later.push_back(l);
                    }
                }
                lanes = first;
                lanes.insert(lanes.end(), later.begin(), later.end());
            }
            int ti = 0;
            for (int l : lanes) dp.thr_tl[ti++] = (int8_t)l;
            for (int l : rest) dp.thr_tl[ti++] = (int8_t)l;
            for (int b = 0; b < k; ++b)  // the run's warp bits, in a fixed order
                if (wb >> b & 1) dp.thr_tl[ti++] = (int8_t)b;

            dp.op_begin = (int)out.ops.size();
            auto rb_of_pos = [&](int p) { return rb_of_tl[tl_of_pos[p]]; };
            for (int li : ph.items) {
                const int gidx = order[sw.items[li]];
                const GateInfo& gi = P.gates[gidx];
                const GateSpec& s = gi.g;
                const int p0 = n - 1 - s.q0;
                const int p1 = gi.nw == 2 ? n - 1 - s.q1 : -1;
                if (adjoint && gi.gen) {
                    DevOp tp{};
                    tp.gate = gidx;
                    tp.moff = -1;
                    tp.tap = ntap++;
                    tp.pos0 = (int8_t)p0;
                    tp.pos1 = (int8_t)p1;
                    tp.rb0 = (int8_t)(tl_of_pos[p0] >= 0 ? rb_of_pos(p0) : -1);
                    tp.rb1 = (int8_t)(p1 >= 0 && tl_of_pos[p1] >= 0 ? rb_of_pos(p1) : -1);
                    tp.kind = gi.gen == 1 ? DK_TX : gi.gen == 2 ? DK_TY : gi.gen == 3 ? DK_TZ : DK_TZZ;
                    out.ops.push_back(tp);
                    out.taps.push_back(DevTap{s.slot, 0, s.coef});
                }
                DevOp op{};
                op.gate = gidx;
                op.tap = -1;
                op.pos0 = (int8_t)p0;
                op.pos1 = (int8_t)p1;
                op.rb0 = (int8_t)(tl_of_pos[p0] >= 0 ? rb_of_pos(p0) : -1);
                op.rb1 = (int8_t)(p1 >= 0 && tl_of_pos[p1] >= 0 ? rb_of_pos(p1) : -1);
                if (gi.diag) {
                    op.kind = gi.nw == 2 ? DK_D2 : DK_D1;
                } else {
                    switch (s.kind) {
                        case QF_H: op.kind = DK_R1; break;
                        case QF_RY: op.kind = DK_RS; break;
                        case QF_RX: op.kind = DK_RX; break;
                        case QF_X: op.kind = DK_X1; break;
                        case QF_CX:
                            op.kind = DK_CX;
                            // target (wire 1) is the register bit, control is pos0
                            op.rb0 = (int8_t)rb_of_pos(p1);
                            op.rb1 = (int8_t)(tl_of_pos[p0] >= 0 ? rb_of_pos(p0) : -1);
                            break;
                        default: op.kind = gi.nw == 2 ? DK_G2 : DK_G1; break;
                    }
                }
                int ms = mat_size(op.kind);
                op.moff = (int16_t)(ms ? moff : -1);
                moff += ms;
                out.ops.push_back(op);
            }
            dp.op_end = (int)out.ops.size();
            out.phases.push_back(dp);
        }
        ds.n_phases = (int)phases.size();
        ds.op_end = (int)out.ops.size();
        ds.n_mat = moff;
        ds.mbase = out.total_mat;
        out.total_mat += (moff + 1) & ~1;  // keep 16-byte alignment of every block
        ds.n_taps = ntap;
        out.n_taps += ntap;
        out.max_mat = std::max(out.max_mat, moff);
        out.max_ops = std::max(out.max_ops, ds.op_end - ds.op_begin);
        out.max_taps = std::max(out.max_taps, ntap);
        out.sweeps.push_back(ds);
    }
}

std::string build_program_plan(int n, const std::vector<GateSpec>& ops, const double* mats,
                               int n_mats, int n_params, int prec, ProgramPlan& P) {
    if (n < 1 || n > 32) return "program: qubit count must be in [1, 32] on the device path";
    if (n_params < 0) return "AnsatzSpec: negative parameter count";
    if (prec != QF_C64 && prec != QF_C128) return "program: precision must be QF_C64 or QF_C128";
    P = ProgramPlan{};
    P.n = n;
    P.prec = prec;
    P.n_params = n_params;
    if (mats && n_mats > 0) P.mats.assign(mats, mats + 32 * (size_t)n_mats);
    P.gates.resize(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) {
        std::string e = classify(n, ops[i], mats, n_mats, n_params, P.gates[i]);
        if (!e.empty()) return e;
        if (ops[i].slot >= 0 && !P.gates[i].gen &&
            (ops[i].kind == QF_SU4 || ops[i].kind == QF_UNITARY)) {
            P.adjoint_ok = false;
            P.adjoint_error = "gradient: parameter feeds a gate without a Pauli generator";
        }
    }
    // commutation DAG (program order among non-commuting gates sharing a wire)
    const int G = (int)ops.size();
    std::vector<std::vector<int>> on_wire(n);
    std::vector<std::vector<int>> preds(G), succs(G);
    for (int j = 0; j < G; ++j) {
        std::set<int> ps;
        for (int w = 0; w < P.gates[j].nw; ++w)
            for (int i : on_wire[P.gates[j].wires[w]])
                if (!commute(P.gates[i], P.gates[j])) ps.insert(i);
        preds[j].assign(ps.begin(), ps.end());
        for (int i : preds[j]) succs[i].push_back(j);
        for (int w = 0; w < P.gates[j].nw; ++w) on_wire[P.gates[j].wires[w]].push_back(j);
    }
    Geometry geo = geometry(prec, n);
    std::vector<int> order(G);
    for (int i = 0; i < G; ++i) order[i] = i;
    lower_pass(P, order, preds, geo.kf, geo.Rf, geo.c, geo.W, false, P.fwd);
    // adjoint: reversed order, reversed DAG
    std::vector<int> rorder(G);
    std::vector<std::vector<int>> rpreds(G);
    for (int i = 0; i < G; ++i) rorder[i] = G - 1 - i;
    for (int i = 0; i < G; ++i) {
        int g = G - 1 - i;
        for (int s : succs[g]) rpreds[i].push_back(G - 1 - s);
    }
    // interleaved complex64 adjoint tiles (QF_JIT_ILV) have 16-byte elements, like
    // complex128: bank groups of 8, so the lane bits are spread mod 3
    const char* ilv = std::getenv("QF_JIT_ILV");  // see jit_interleaved (jit.cpp)
    const int Wb = (prec == QF_C64 && ilv && ilv[0] == '1') ? 3 : geo.W;
    lower_pass(P, rorder, rpreds, geo.kb, geo.Rb, geo.c, Wb, true, P.bwd);
    if (G > 0 && (P.fwd.sweeps.empty() || P.bwd.sweeps.empty()))
        return "program: scheduling failed";
    return "";
}

std::string build_observable_plan(int n, int n_terms, const int8_t* codes, const double* w_re,
                                  const double* w_im, int kh, ObservablePlan& O) {
    if (n < 1 || n > 32) return "observable: qubit count must be in [1, 32] on the device path";
    if (n_terms < 0) return "observable: negative term count";
    O = ObservablePlan{};
    O.n = n;
    O.kh = kh;
    const uint32_t lo = (kh >= 32) ? 0xffffffffu : ((1u << kh) - 1);
    std::map<uint32_t, std::vector<DevTerm>> groups;
    groups[0];  // own tile always first (energy needs it)
    for (int t = 0; t < n_terms; ++t) {
        uint32_t flip = 0, z = 0;
        int y = 0;
        for (int i = 0; i < n; ++i) {  // compile_term, pauli.cpp:61-74
            int c = codes[(size_t)t * n + i];
            if (c < 0 || c > 3) return "PauliSum::add: code out of range";
            uint32_t bit = 1u << (n - 1 - i);
            if (c == 1) flip |= bit;
            if (c == 2) { flip |= bit; z |= bit; ++y; }
            if (c == 3) z |= bit;
        }
        if (!std::isfinite(w_re[t]) || !std::isfinite(w_im ? w_im[t] : 0.0))
            return "PauliSum::add: non-finite weight";
        static const double ip[4][2] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
        DevTerm d{};
        const double wr = w_re[t], wi = w_im ? w_im[t] : 0.0;
        d.c_re = wr * ip[y & 3][0];
        d.c_im = wr * ip[y & 3][1];
        d.ci_re = wi * ip[y & 3][0];
        d.ci_im = wi * ip[y & 3][1];
        if (wi != 0.0) O.has_imag = true;
        d.f_in = flip & lo;
        d.z = z;
        d.fz_par = (uint32_t)(__builtin_popcount(flip & z) & 1);
        d.yodd = y & 1;
        d.kind = flip == 0 ? TK_DIAG : (z == 0 ? TK_FLIP : TK_GEN);
        groups[flip & ~lo].push_back(d);
    }
    for (auto& [fo, ts] : groups) {
        DevGroup g{};
        g.f_out = fo;
        g.term_begin = (int)O.terms.size();
        // diagonal terms first, then pure flips, then general (kernel loops per kind)
        for (int kind = 0; kind < 3; ++kind)
            for (auto& d : ts)
                if (d.kind == kind) O.terms.push_back(d);
        g.term_end = (int)O.terms.size();
        O.groups.push_back(g);
    }
    return "";
}

}  // namespace qfb
