// planner.cpp -- per-trajectory program construction.
//
//  1. Alg. 2 first loop for every channel: one Philox draw per
//     channel; r < cumulative pbar picks K_i and DEFERS it (it becomes an
//     ordinary operation for the fuser); otherwise the channel is
//     CONVENTIONAL (a barrier: every earlier operation is applied, then rho_Q
//     is reduced on the device and lines 13-21 pick K_i there).
//  2. Each barrier-free segment is fused with the paper's two-phase fuser
//     (Sec. III.B) at maximum fuse size f.
//  3. Fused gates are packed greedily into tile passes: a pass holds <= T
//     qubits (the CL lowest always included), so one HBM read + write applies
//     many fused gates (the B200 design; the paper applies one fused gate per
//     sweep, which one_gate_per_pass reproduces).
//  4. Epilogues: rho_Q at each barrier; block sums (+ Pauli partials) at the
//     end of the trajectory.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "host.hpp"
#include "philox.hpp"

namespace qt {

static inline int popc(uint64_t x) { return __builtin_popcountll(x); }

// ---------------------------------------------------------------------------
// Two-phase fuser.  Flat arrays in a per-thread scratch (planning runs
// per trajectory on every host thread; no heap traffic in steady state).
// ---------------------------------------------------------------------------
namespace {
struct FuseScratch {
    std::vector<int> qcnt, qoff, onq, slot;         // per-qubit item lists (CSR), item slots (6 per item)
    std::vector<int> group, gid, anchor;            // phase 1 groups
    std::vector<char> absorbed, has_members;
    std::vector<int> moff, mem;                     // members per group (CSR, time order)
    std::vector<uint64_t> gmask;
    std::vector<char> gfixed, marked;
    std::vector<int> gqcnt, gqoff, gq, gpos;        // per-qubit group lists (CSR), group slots (6 per group)
    std::vector<int> F, last;                       // phase 2 growth
};
template <class V>
inline void fit(V& v, size_t n) {
    if (v.size() < n) v.resize(n);
}
}  // namespace

#ifdef QT_PLAN_PROFILE
// diagnostics build: seconds spent per planning phase (single-threaded callers)
static double g_prof[8];
extern "C" void qt_plan_profile(double* o) {
    for (int i = 0; i < 8; ++i) o[i] = g_prof[i];
}
#define QT_PP(k)                                                                                      \
    do {                                                                                              \
        const auto t_now = std::chrono::steady_clock::now();                                          \
        g_prof[k] += std::chrono::duration<double>(t_now - t_pp).count();                             \
        t_pp = t_now;                                                                                 \
    } while (0)
#else
#define QT_PP(k)
#endif

void fuse_items(const FuseItem* items, int N, int f, std::vector<int>& flat, std::vector<int>& offs) {
#ifdef QT_PLAN_PROFILE
    auto t_pp = std::chrono::steady_clock::now();
#endif
    flat.clear();
    offs.assign(1, 0);
    if (N == 0) return;
    thread_local FuseScratch S;
    int nq = 0;
    for (int i = 0; i < N; ++i) nq = std::max(nq, 64 - __builtin_clzll(items[i].mask | 1));
    // per-qubit item sequences (CSR) and each item's slot in them
    fit(S.qcnt, nq);
    fit(S.qoff, nq + 1);
    std::fill(S.qcnt.begin(), S.qcnt.begin() + nq, 0);
    for (int i = 0; i < N; ++i)
        for (uint64_t mk = items[i].mask; mk; mk &= mk - 1) ++S.qcnt[__builtin_ctzll(mk)];
    S.qoff[0] = 0;
    for (int q = 0; q < nq; ++q) S.qoff[q + 1] = S.qoff[q] + S.qcnt[q];
    fit(S.onq, S.qoff[nq]);
    fit(S.slot, 6 * (size_t)N);
    std::fill(S.qcnt.begin(), S.qcnt.begin() + nq, 0);
    for (int i = 0; i < N; ++i) {
        int m = 0;
        for (uint64_t mk = items[i].mask; mk; mk &= mk - 1, ++m) {
            const int q = __builtin_ctzll(mk);
            S.slot[6 * i + m] = S.qcnt[q];
            S.onq[S.qoff[q] + S.qcnt[q]++] = i;
        }
    }
    auto onq = [&](int q, int k) { return S.onq[S.qoff[q] + k]; };
    // ---- phase 1: absorb small items into time-adjacent larger ones on the same qubits
    fit(S.group, N);
    fit(S.absorbed, N);
    fit(S.has_members, N);
    int* group = S.group.data();
    for (int i = 0; i < N; ++i) {
        group[i] = i;
        S.absorbed[i] = 0;
        S.has_members[i] = 0;
    }
    auto kq = [&](int g) { return popc(items[g].mask); };
    // forward absorption (an item joins the next larger item on all of its qubits); reverse order
    for (int i = N - 1; i >= 0; --i) {
        if (items[i].fixed) continue;
        int G = -1;
        bool ok = true;
        int m = 0;
        for (uint64_t mk = items[i].mask; mk && ok; mk &= mk - 1, ++m) {
            const int q = __builtin_ctzll(mk);
            const int pos = S.slot[6 * i + m];
            if (pos + 1 >= S.qcnt[q]) { ok = false; break; }
            const int g = group[onq(q, pos + 1)];
            if (G < 0) G = g;
            else if (G != g) ok = false;
        }
        if (!ok || G < 0 || items[G].fixed) continue;
        if (!((items[i].mask & ~items[G].mask) == 0 && popc(items[i].mask) < kq(G))) continue;
        group[i] = G;
        S.absorbed[i] = 1;
    }
    // backward absorption of trailing small items into the previous larger item
    for (int i = 0; i < N; ++i)
        if (group[i] != i) S.has_members[group[i]] = 1;
    for (int i = 0; i < N; ++i) {
        if (items[i].fixed || S.absorbed[i] || S.has_members[i]) continue;
        int G = -1;
        bool ok = true;
        int m = 0;
        for (uint64_t mk = items[i].mask; mk && ok; mk &= mk - 1, ++m) {
            const int q = __builtin_ctzll(mk);
            const int pos = S.slot[6 * i + m];
            if (pos == 0) { ok = false; break; }
            const int g = group[onq(q, pos - 1)];
            if (G < 0) G = g;
            else if (G != g) ok = false;
        }
        if (!ok || G < 0 || items[G].fixed) continue;
        if (!((items[i].mask & ~items[G].mask) == 0 && popc(items[i].mask) < kq(G))) continue;
        group[i] = G;
        S.absorbed[i] = 1;
        S.has_members[G] = 1;
    }
    QT_PP(6);
    // groups in anchor order (rank = group id); members in time order
    fit(S.gid, N);
    int G = 0;
    for (int i = 0; i < N; ++i)
        if (group[i] == i) S.gid[i] = G++;
    fit(S.gmask, N);
    fit(S.gfixed, N);
    fit(S.moff, N + 1);
    fit(S.mem, N);
    auto build_groups = [&](bool phase1) {
        if (!phase1) {
            G = N;
            for (int i = 0; i < N; ++i) S.gid[i] = i;
        }
        std::fill(S.moff.begin(), S.moff.begin() + G + 1, 0);
        for (int i = 0; i < N; ++i) {
            const int a = phase1 ? group[i] : i;
            ++S.moff[S.gid[a] + 1];
            if (a == i) {
                S.gmask[S.gid[i]] = items[i].mask;
                S.gfixed[S.gid[i]] = items[i].fixed;
            }
        }
        for (int g = 0; g < G; ++g) S.moff[g + 1] += S.moff[g];
        fit(S.last, G);
        for (int g = 0; g < G; ++g) S.last[g] = S.moff[g];
        for (int i = 0; i < N; ++i) S.mem[S.last[S.gid[phase1 ? group[i] : i]]++] = i;
        // per-qubit group sequences (dedup consecutive); valid iff strictly increasing rank
        fit(S.gqcnt, nq);
        fit(S.gqoff, nq + 1);
        fit(S.gq, S.qoff[nq]);
        bool valid = true;
        for (int q = 0; q < nq; ++q) {
            int c = 0;
            const int base = S.qoff[q];
            for (int k = 0; k < S.qcnt[q]; ++k) {
                const int g = S.gid[phase1 ? group[onq(q, k)] : onq(q, k)];
                if (c == 0 || S.gq[base + c - 1] != g) {
                    if (c > 0 && S.gq[base + c - 1] >= g) valid = false;
                    S.gq[base + c++] = g;
                }
            }
            S.gqcnt[q] = c;
            S.gqoff[q] = base;
        }
        return valid;
    };
    if (!build_groups(true)) build_groups(false);  // fall back: no phase-1 absorption
    // position of each group in each of its qubits' group lists
    fit(S.gpos, 6 * (size_t)G);
    for (int q = 0; q < nq; ++q)
        for (int k = 0; k < S.gqcnt[q]; ++k) {
            const int g = S.gq[S.gqoff[q] + k];
            int m = 0;
            for (uint64_t mk = S.gmask[g]; mk; mk &= mk - 1, ++m)
                if (__builtin_ctzll(mk) == q) S.gpos[6 * g + m] = k;
        }
    auto pos_on = [&](int g, int q) {
        int m = 0;
        for (uint64_t mk = S.gmask[g]; mk; mk &= mk - 1, ++m)
            if (__builtin_ctzll(mk) == q) return S.gpos[6 * g + m];
        return -1;
    };
    auto gqat = [&](int q, int k) { return S.gq[S.gqoff[q] + k]; };
    QT_PP(7);
    // ---- phase 2: greedy growth in increasing time order
    fit(S.marked, G);
    std::fill(S.marked.begin(), S.marked.begin() + G, 0);
    char* marked = S.marked.data();
    auto ready = [&](int h) {  // all predecessors of h marked
        int m = 0;
        for (uint64_t mk = S.gmask[h]; mk; mk &= mk - 1, ++m) {
            const int q = __builtin_ctzll(mk);
            const int p = S.gpos[6 * h + m];
            if (p > 0 && !marked[gqat(q, p - 1)]) return false;
        }
        return true;
    };
    fit(S.last, (size_t)std::max(nq, 1));
    flat.reserve(N);
    offs.reserve(G + 1);
    for (int g0 = 0; g0 < G; ++g0) {
        if (marked[g0]) continue;
        S.F.clear();
        S.F.push_back(g0);
        marked[g0] = 1;
        uint64_t FM = S.gmask[g0];
        // last[q]: latest position of a member of F on qubit q (q in FM)
        {
            int m = 0;
            for (uint64_t mk = FM; mk; mk &= mk - 1, ++m) S.last[__builtin_ctzll(mk)] = S.gpos[6 * g0 + m];
        }
        uint64_t cur = FM;  // qubits whose last[] is set
        auto add_group = [&](int g) {
            marked[g] = 1;
            S.F.push_back(g);
            int m = 0;
            for (uint64_t mk = S.gmask[g]; mk; mk &= mk - 1, ++m) {
                const int q = __builtin_ctzll(mk);
                const int p = S.gpos[6 * g + m];
                if (!((cur >> q) & 1) || p > S.last[q]) S.last[q] = p;
            }
            cur |= S.gmask[g];
        };
        if (!S.gfixed[g0]) {
            bool added = true;
            while (added) {
                added = false;
                for (uint64_t mk = FM; mk; mk &= mk - 1) {
                    const int q = __builtin_ctzll(mk);
                    // the next group on q after F's latest member there
                    const int lq = S.last[q];
                    if (lq + 1 >= S.gqcnt[q]) continue;
                    const int h = gqat(q, lq + 1);
                    if (marked[h] || S.gfixed[h]) continue;
                    // unmarked predecessors of h (next-nearest neighbours back in time)
                    int preds[6], np = 0;
                    bool ok = true;
                    uint64_t nm = FM | S.gmask[h];
                    int m = 0;
                    for (uint64_t hm = S.gmask[h]; hm && ok; hm &= hm - 1, ++m) {
                        const int p = __builtin_ctzll(hm);
                        const int ph = S.gpos[6 * h + m];
                        if (ph <= 0) continue;
                        const int pg = gqat(p, ph - 1);
                        if (marked[pg]) continue;
                        if (S.gfixed[pg] || !ready(pg)) { ok = false; break; }
                        bool seen = false;
                        for (int j = 0; j < np; ++j) seen |= preds[j] == pg;
                        if (!seen) {
                            preds[np++] = pg;
                            nm |= S.gmask[pg];
                        }
                    }
                    if (!ok || popc(nm) > f) continue;
                    for (int j = 0; j < np; ++j) add_group(preds[j]);
                    add_group(h);
                    FM = nm;
                    added = true;
                    break;  // restart from the lowest qubit with the grown set
                }
            }
        }
        std::sort(S.F.begin(), S.F.end());
        for (int g : S.F)
            for (int k = S.moff[g]; k < S.moff[g + 1]; ++k) flat.push_back(S.mem[k]);
        offs.push_back((int)flat.size());
    }
}

// ---------------------------------------------------------------------------
// Pass building.
// ---------------------------------------------------------------------------
namespace {

struct FusedGate {
    uint64_t mask;
    const int* items;  // indices into the segment item list (the fuser's flat output)
    int n_items;
    int special_event;  // >= 0: device-chosen conventional op (no materialization)
    const int* begin() const { return items; }
    const int* end() const { return items + n_items; }
};

struct Item {
    uint64_t mask;
    int var;      // variant, or -1 for the device-chosen op
    int event;    // event index for the device-chosen op
    int nq;
};

inline uint64_t low_mask(int k) { return k >= 64 ? ~0ull : ((1ull << k) - 1ull); }

uint64_t fill_tile(uint64_t S, int T, int n) {
    for (int q = 0; q < n && popc(S) < T; ++q) S |= 1ull << q;
    return S;
}

// Register layout of a fused gate inside a tile (see GateDesc): register bits
// 0..k-1 = the gate's tile-local bits ascending, k..R-1 = the highest other
// tile bits (so the lane bits stay low: bank-conflict-free re-layouts),
// thread bits = the remaining tile bits ascending.
void gate_layout(uint64_t gate_mask, uint64_t S, int T, int R, uint32_t& rpos, uint32_t& tpos) {
    uint32_t regmask = 0;
    rpos = 0;
    int m = 0;
    for (uint64_t mk = gate_mask; mk; mk &= mk - 1, ++m) {
        const int q = __builtin_ctzll(mk);
        const int p = popc(S & low_mask(q));
        rpos |= (uint32_t)p << (4 * m);
        regmask |= 1u << p;
    }
    for (int p = T - 1; p >= 0 && m < R; --p)
        if (!((regmask >> p) & 1u)) {
            rpos |= (uint32_t)p << (4 * m);
            regmask |= 1u << p;
            ++m;
        }
    tpos = 0;
    int i = 0;
    for (int p = 0; p < T; ++p)
        if (!((regmask >> p) & 1u)) tpos |= (uint32_t)p << (4 * i++);
}

// Byte offset of tile bit b in the f16 operand layout of a 4-qubit tensor-core
// gate (tile_pass_kernel.cuh a_offset): matrix bit m -> 8 << m, group bit
// (rpos[4]) -> 16 KB, thread bit i -> row bit i of the SWIZZLE_128B layout.
uint32_t operand_unit(const GateDesc& gd, int b) {
    for (int m = 0; m < 5; ++m)
        if ((int)((gd.rpos >> (4 * m)) & 15u) == b) return m < 4 ? 8u << m : 16384u;
    for (int i = 0; i < 7; ++i)
        if ((int)((gd.tpos >> (4 * i)) & 15u) == b) return i < 3 ? ((128u << i) ^ (16u << i)) : (128u << i);
    return 0;
}

// Bank vector (shared-memory address bits 3..6 of an 8-byte amplitude) of tile
// bit b in the layout a gate's outputs are written to: the next gate's f16
// operand layout (matrix bit m -> address bit 3 + m, thread bit i < 3 -> address
// bit 4 + i, other roles leave the bank unchanged) or, with nx == nullptr, the
// swizzled fp32 tile (tile bit b -> swizzle bit b mod 4).
unsigned bank_vec(const GateDesc* nx, int b) {
    if (!nx) return 1u << (b & 3);
    for (int m = 0; m < 4; ++m)
        if ((int)((nx->rpos >> (4 * m)) & 15u) == b) return 1u << m;
    for (int i = 0; i < 3; ++i)
        if ((int)((nx->tpos >> (4 * i)) & 15u) == b) return 2u << i;
    return 0;
}

// Thread-bit order of a tensor-core gate: the four lowest thread bits (a
// half-warp's lanes) get tile bits whose bank vectors in the output layout are
// linearly independent, so the half-warp's 8-byte stores of one configuration
// hit 16 distinct bank pairs; the group bit is the highest remaining tile bit.
// GF(2) rank of up to 4 bank vectors (4-bit).
int rank4(const unsigned* v, int count) {
    unsigned basis[4] = {0, 0, 0, 0};
    int r = 0;
    for (int i = 0; i < count; ++i) {
        unsigned x = v[i];
        for (int j = 3; j >= 0 && x; --j)
            if ((x >> j) & 1u) {
                if (!basis[j]) {
                    basis[j] = x;
                    ++r;
                    break;
                }
                x ^= basis[j];
            }
    }
    return r;
}

// run_start: the gate also gathers the fp32 tile in its layout at the start of
// the run (8-byte loads, bank vector of tile bit b = 2^(b mod 4) under the
// tile swizzle), so the four lane bits are chosen among all subsets of the
// free tile bits: full rank for the stores first, then for the gather.
void tc_relayout(GateDesc& gd, const GateDesc* nx, int T, int grp, bool run_start = false) {
    uint32_t cfg = 0;
    for (int m = 0; m < 4; ++m) cfg |= 1u << ((gd.rpos >> (4 * m)) & 15u);
    if (gd.pair) {
        // paired 16-byte stores: a quarter-warp's 8 lanes must hit 8 distinct chunks
        // (address bits 4..6: bank vectors without bit 0); among those choices the
        // run-start fp32 gather (4 lanes, 2^(b mod 4)) decides
        int cand[12], nc = 0;
        for (int b = 0; b < T; ++b)
            if (!(((cfg | (1u << grp)) >> b) & 1u)) cand[nc++] = b;
        int best[4] = {-1, -1, -1, -1}, best_score = -1;
        for (int a = 0; a < nc; ++a)
            for (int b = 0; b < nc; ++b)
                for (int c = 0; c < nc; ++c)
                    for (int d = 0; d < nc; ++d) {
                        if (b <= a || c <= b || a == d || b == d || c == d) continue;  // lanes 0-2 ascending, lane 3 any
                        const int pick[4] = {cand[a], cand[b], cand[c], cand[d]};
                        unsigned vs[3], vg[4];
                        for (int i = 0; i < 3; ++i) vs[i] = bank_vec(nx, pick[i]) >> 1;
                        for (int i = 0; i < 4; ++i) vg[i] = 1u << (pick[i] & 3);
                        const int score = 8 * rank4(vs, 3) + (run_start ? rank4(vg, 4) : 0);
                        if (score > best_score) {
                            best_score = score;
                            for (int i = 0; i < 4; ++i) best[i] = pick[i];
                        }
                    }
        if (best_score >= 0) {
            int lanes[12], nl = 0;
            uint32_t used = cfg | (1u << grp);
            for (int i = 0; i < 4; ++i) {
                lanes[nl++] = best[i];
                used |= 1u << best[i];
            }
            for (int b = 0; b < T; ++b)
                if (!((used >> b) & 1u)) lanes[nl++] = b;
            gd.rpos = (gd.rpos & 0xffffu) | ((uint32_t)grp << 16);
            gd.tpos = 0;
            for (int i = 0; i < nl; ++i) gd.tpos |= (uint32_t)lanes[i] << (4 * i);
            return;
        }
    }
    if (run_start) {
        int cand[12], nc = 0;
        for (int b = 0; b < T; ++b)
            if (!(((cfg | (1u << grp)) >> b) & 1u)) cand[nc++] = b;
        int best[4] = {-1, -1, -1, -1}, best_score = -1;
        for (int a = 0; a < nc; ++a)
            for (int b = a + 1; b < nc; ++b)
                for (int c = b + 1; c < nc; ++c)
                    for (int d = c + 1; d < nc; ++d) {
                        const int pick[4] = {cand[a], cand[b], cand[c], cand[d]};
                        unsigned vs[4], vg[4];
                        for (int i = 0; i < 4; ++i) {
                            vs[i] = bank_vec(nx, pick[i]);
                            vg[i] = 1u << (pick[i] & 3);
                        }
                        const int score = 8 * rank4(vs, 4) + rank4(vg, 4);
                        if (score > best_score) {
                            best_score = score;
                            for (int i = 0; i < 4; ++i) best[i] = pick[i];
                        }
                    }
        if (best_score >= 0) {
            int lanes[12], nl = 0;
            uint32_t used = cfg | (1u << grp);
            for (int i = 0; i < 4; ++i) {
                lanes[nl++] = best[i];
                used |= 1u << best[i];
            }
            for (int b = 0; b < T; ++b)
                if (!((used >> b) & 1u)) lanes[nl++] = b;
            gd.rpos = (gd.rpos & 0xffffu) | ((uint32_t)grp << 16);
            gd.tpos = 0;
            for (int i = 0; i < nl; ++i) gd.tpos |= (uint32_t)lanes[i] << (4 * i);
            return;
        }
    }
    int lanes[12], nl = 0;
    unsigned basis[4] = {0, 0, 0, 0};  // GF(2) basis by leading bit
    uint32_t used = cfg | (1u << grp);
    for (int b = 0; b < T && nl < 4; ++b) {
        if ((used >> b) & 1u) continue;
        unsigned v = bank_vec(nx, b);
        for (int j = 3; j >= 0 && v; --j)
            if ((v >> j) & 1u) {
                if (!basis[j]) {
                    basis[j] = v;
                    break;
                }
                v ^= basis[j];
            }
        if (!v) continue;
        lanes[nl++] = b;
        used |= 1u << b;
    }
    for (int b = 0; b < T; ++b)
        if (!((used >> b) & 1u)) lanes[nl++] = b;
    gd.rpos = (gd.rpos & 0xffffu) | ((uint32_t)grp << 16);
    gd.tpos = 0;
    for (int i = 0; i < nl; ++i) gd.tpos |= (uint32_t)lanes[i] << (4 * i);
}

// Tensor-core runs of one pass (desc.hpp GateDesc): a run starts at the first
// tensor-core gate, after a CUDA-core gate, or when the product of the runs'
// norm bounds would exceed 16 (the f16 tile scale has 2^2.5 headroom beyond
// contractions, widened by 2^shift); layouts are chosen last gate first for
// conflict-free stores into the next layout; xu = next-gate operand offsets
// of this gate's roles when the run continues.
void tc_runs(GateDesc* gd, const double* norms, int count, int T, std::vector<FusedDesc>& fused,
             std::vector<ConsDesc>& cons, const int* gate_fused) {
    auto cfg_of = [&](int g) {
        uint32_t c = 0;
        for (int m = 0; m < 4; ++m) c |= 1u << ((gd[g].rpos >> (4 * m)) & 15u);
        return c;
    };
    int first = -1;
    double cum = 1.0;
    const uint32_t all = (1u << T) - 1u;
    for (int g = 0; g < count; ++g) {
        if (!(gd[g].k & kGateTC)) {
            first = -1;
            continue;
        }
        if (first < 0 || cum * norms[g] > 16.0) {
            first = g;
            cum = 1.0;
            gd[g].k |= kGateRunStart;
        }
        cum *= norms[g];
        const int shift = cum > 1.0 ? std::min(100, (int)std::ceil(std::log2(cum))) : 0;
        gd[first].k = (gd[first].k & ~(0xff << kGateShiftBit)) | (shift << kGateShiftBit);
    }
    auto chained = [&](int g) {
        return g + 1 < count && (gd[g].k & kGateTC) && (gd[g + 1].k & (kGateTC | kGateRunStart)) == kGateTC;
    };
    // runs of one gate keep the 3xTF32 path (no operand-layout conversion)
    for (int g = 0; g < count; ++g)
        if ((gd[g].k & kGateTC) && (chained(g) || (g > 0 && chained(g - 1)))) gd[g].k |= kGateF16;
    // group bit: runs are cut into maximal segments whose gates leave a common
    // tile bit untouched; that bit is the segment's group bit, so inside a
    // segment the two 128-row groups pipeline independently (K1 tc_run_f16)
    std::vector<int> grp(count, -1);
    for (int g = 0; g < count;) {
        if (!(gd[g].k & kGateF16)) {
            ++g;
            continue;
        }
        int e = g;
        uint32_t u = cfg_of(g);
        while (chained(e) && (u | cfg_of(e + 1)) != all) u |= cfg_of(++e);
        int b = T - 1;
        while (b >= 0 && ((u >> b) & 1u)) --b;
        for (int x = g; x <= e; ++x) grp[x] = b;
        g = e + 1;
    }
    for (int g = count - 1; g >= 0; --g) {
        if (!(gd[g].k & kGateF16)) continue;
        gd[g].pair = 0;
        if (chained(g) && gate_fused[g] >= 0) {
            // the next gate's matrix bit 0 is address bit 3 (the 8-byte half of a
            // chunk): if it is one of this gate's matrix bits m0, relabel this gate's
            // matrix bits 0 <-> m0 (register order and its constituents' positions,
            // so K6 builds W in that order); outputs c, c ^ 1 then share a chunk
            const uint32_t t0 = gd[g + 1].rpos & 15u;
            int m0 = -1;
            for (int m = 0; m < 4; ++m)
                if (((gd[g].rpos >> (4 * m)) & 15u) == t0) m0 = m;
            if (m0 > 0) {
                const uint32_t r0 = gd[g].rpos & 15u, rm = (gd[g].rpos >> (4 * m0)) & 15u;
                gd[g].rpos = (gd[g].rpos & ~(15u | (15u << (4 * m0)))) | rm | (r0 << (4 * m0));
                const FusedDesc& fd = fused[gate_fused[g]];
                for (int ci = fd.cons_begin; ci < fd.cons_begin + fd.cons_count; ++ci) {
                    uint32_t pos = cons[ci].pos;
                    // K6 reads the first nq (<= 6) nibbles; the others are ignored
                    for (int j = 0; j < 6; ++j) {
                        const uint32_t p = (pos >> (4 * j)) & 15u;
                        const uint32_t q = p == 0u ? (uint32_t)m0 : (p == (uint32_t)m0 ? 0u : p);
                        pos = (pos & ~(15u << (4 * j))) | (q << (4 * j));
                    }
                    cons[ci].pos = pos;
                }
            }
            if (m0 >= 0) gd[g].pair = 1;
        }
        tc_relayout(gd[g], chained(g) ? &gd[g + 1] : nullptr, T, grp[g], !(g > 0 && chained(g - 1)));
    }
    for (int g = 0; g < count; ++g) {
        if (!chained(g)) continue;
        for (int r = 0; r < 12; ++r) {
            const int b = r < 5 ? (int)((gd[g].rpos >> (4 * r)) & 15u) : (int)((gd[g].tpos >> (4 * (r - 5))) & 15u);
            gd[g].xu[r] = (uint16_t)operand_unit(gd[g + 1], b);
        }
    }
}

// Persistent TMEM kernel layouts (tile_pass_v2.cu, T = 13).  A fused 4-qubit gate
// is one M128 x N32 x K96 real GEMM per group: 7 tile bits index the 128 TMEM lanes
// (rows), 2 are group bits (four D / A column blocks per thread) and its 4 matrix
// bits are the columns.  Consecutive gates whose qubits, together, fit in 6 tile
// bits form a SEGMENT with one row set: between them the epilogue reads D and
// writes the next A inside TMEM (each thread keeps its row; only the roles of the
// 6 thread-local bits change), with the next gate's source columns xu.  A segment
// starts by gathering the fp32 tile from shared memory and ends by writing it back.
namespace {
inline unsigned v2_bank(int b) {  // slot bits 0..3 of tile bit b under the T = 13 swizzle
    if (b == 0) return 1u;
    if (b < 4) return 1u << b;
    return 2u << ((b - 4) % 3);
}
}  // namespace

// TMA-pipelined kernel (tile_pass_v3.cu, T = 11): the 7 thread bits (tpos) of a gate,
// reordered so that a warp's lanes reach distinct shared-memory banks under the TMA
// SWIZZLE_128B image (tile bit b -> 8-byte bank-pair bit b for b < 4, bits 4..6 fold onto
// pair bits 1..3, bits >= 7 none): 16-byte pair accesses (matrix bit 0 = tile bit 0) are
// served per quarter warp (lanes 0..2 must cover pair bits 1, 2, 3), 8-byte accesses per
// half warp (lanes 0..3: pair bits 0..3).
void v3_lanes(GateDesc& gd) {
    int rows[7], nr = 0;
    for (int i = 0; i < 7; ++i) rows[nr++] = (int)((gd.tpos >> (4 * i)) & 15u);
    const bool pair = (gd.k & kGateTC) && (gd.rpos & 15u) == 0u;
    bool used[7] = {false, false, false, false, false, false, false};
    int order[7], no = 0;
    auto take = [&](int b) {
        for (int i = 0; i < 7; ++i)
            if (!used[i] && rows[i] == b) {
                used[i] = true;
                order[no++] = b;
                return true;
            }
        return false;
    };
    if (!pair) take(0);
    for (int c = 1; c <= 3; ++c)
        if (!take(c)) take(c + 3);
    for (int i = 0; i < 7; ++i)
        if (!used[i]) {
            used[i] = true;
            order[no++] = rows[i];
        }
    gd.tpos = 0;
    for (int i = 0; i < 7; ++i) gd.tpos |= (uint32_t)order[i] << (4 * i);
    // swizzled byte offsets of the roles for the kernel: xu[0..3] register / matrix bits
    // (rpos), xu[4..10] thread bits (tpos)
    auto swzb = [](int b) { const uint32_t x = 8u << b; return (uint16_t)(x ^ (((x >> 7) & 7u) << 4)); };
    for (int m = 0; m < 4; ++m) gd.xu[m] = swzb((int)((gd.rpos >> (4 * m)) & 15u));
    for (int i = 0; i < 7; ++i) gd.xu[4 + i] = swzb(order[i]);
}

// Layout roles of a v2 gate: the tile bits of its matrix bits (cfg, in matrix-bit
// order), of its two group bits, of the 5 TMEM lane bits and of the 2 warp bits.
struct V2Lay {
    int cfg[4], grp[2], lane[5], warp[2];
};

void v2_layouts(GateDesc* gd, const uint32_t* lmask, const double* norms, int count, std::vector<FusedDesc>& fused,
                std::vector<ConsDesc>& cons, const int* gate_fused) {
    constexpr int T = 13;
    constexpr int kNever = 1 << 20;
    static const bool half_split = getenv("QT_V2_HALF") && atoi(getenv("QT_V2_HALF")) != 0;
    auto bits_of = [](uint32_t m, int* out) {
        int k = 0;
        for (int b = 0; b < 13; ++b)
            if ((m >> b) & 1u) out[k++] = b;
        return k;
    };
    // first gate index > i that uses tile bit b (tensor-core gates of this pass), from a
    // table filled by one backward scan
    thread_local std::vector<int> nu_tab;
    if (nu_tab.size() < (size_t)13 * (count + 1)) nu_tab.resize((size_t)13 * (count + 1));
    for (int b = 0; b < 13; ++b) nu_tab[(size_t)13 * count + b] = kNever;
    for (int j = count - 1; j >= 0; --j)
        for (int b = 0; b < 13; ++b) {
            // entry j: next use after gate j - 1 ... stored as "first index >= j"
            int v;
            if (!(gd[j].k & kGateTC)) v = kNever;
            else if ((lmask[j] >> b) & 1u) v = j;
            else v = nu_tab[(size_t)13 * (j + 1) + b];
            nu_tab[(size_t)13 * j + b] = v;
        }
    auto next_use = [&](int i, int b) { return nu_tab[(size_t)13 * (i + 1) + b]; };
    // matrix-bit order of gate i's qubits: `first` (or -1) fixed at bit 0, then the
    // qubits needed latest at bits 0 / 1 (they leave for lane bits at an X transition),
    // the ones needed soonest at bits 2 / 3
    auto order_cfg = [&](int i, int first, int* cfg) {
        int q[4];
        bits_of(lmask[i], q);
        int rest[4], nr = 0;
        for (int t = 0; t < 4; ++t)
            if (q[t] != first) rest[nr++] = q[t];
        std::stable_sort(rest, rest + nr, [&](int a, int b) { return next_use(i, a) > next_use(i, b); });
        int m = 0;
        if (first >= 0) cfg[m++] = first;
        for (int t = 0; t < nr; ++t) cfg[m++] = rest[t];
    };
    // tile bit 0 as matrix bit 0 (16-byte pair gathers / write-backs, kGatePair0) when
    // it is one of the two bits leaving at the next X transition anyway
    auto pair0 = [](V2Lay& L) {
        if (L.cfg[1] == 0) std::swap(L.cfg[0], L.cfg[1]);
    };
    // modelled shared-memory wavefronts per 8 bytes of a warp's fp32-tile access with
    // this layout (2 = conflict-free): 16-byte pair accesses are served per quarter warp
    // (lane bits 0..2 must reach 8 distinct 16-byte chunks), 8-byte ones per half warp
    // (lane bits 0..3 must reach the 16 bank pairs)
    auto wf8 = [](const V2Lay& L) {
        const int nl = L.cfg[0] == 0 ? 3 : 4;
        unsigned basis[4];
        int r = 0;
        for (int t = 0; t < nl; ++t) {
            unsigned v = v2_bank(L.lane[t]);
            for (int j = 0; j < r; ++j) v = std::min(v, v ^ basis[j]);
            if (v) basis[r++] = v;
        }
        return 2 << (nl - r);
    };
    // fresh layout of gate i (segment start: gathered from the fp32 tile)
    auto fresh = [&](int i, V2Lay& L) {
        order_cfg(i, -1, L.cfg);
        // tile bits not in gate i, in order of next use
        int fut[13], nf = 0;
        for (int b = 0; b < T; ++b)
            if (!((lmask[i] >> b) & 1u)) fut[nf++] = b;
        std::stable_sort(fut, fut + nf, [&](int a, int b) { return next_use(i, a) < next_use(i, b); });
        // group bits: the two needed soonest (local transitions); then lane bits by
        // arrival through X transitions (L3, L4 next, L1, L2 after one X, L0 after
        // two); the bits never needed are warp bits
        static const int lane_order[5] = {3, 4, 1, 2, 0};
        if (half_split) {
            // group bit 1 selects the warpgroup half and stays for the whole segment:
            // with the warp bits it takes the three bits needed last
            L.grp[0] = fut[0];
            for (int t = 0; t < 5; ++t) L.lane[lane_order[t]] = fut[1 + t];
            L.warp[0] = fut[6];
            L.warp[1] = fut[7];
            L.grp[1] = fut[8];
        } else {
            L.grp[0] = fut[0];
            L.grp[1] = fut[1];
            for (int t = 0; t < 5; ++t) L.lane[lane_order[t]] = fut[2 + t];
            L.warp[0] = fut[7];
            L.warp[1] = fut[8];
        }
        pair0(L);
        // conflict-free gathers: swap lane bits 0..2 with the warp bits (the tile bits
        // needed last) when that lowers the modelled wavefronts, lane bit 0 first
        int best = wf8(L);
        V2Lay B = L;
        static const int lpos[3] = {0, 2, 1};
        for (int a = 0; a < 3 && best > 2; ++a)
            for (int w = 0; w < 2; ++w) {
                V2Lay X = L;
                std::swap(X.lane[lpos[a]], X.warp[w]);
                const int f = wf8(X);
                if (f < best) {
                    best = f;
                    B = X;
                }
            }
        for (int a = 0; a < 3 && best > 2; ++a)
            for (int b = a + 1; b < 3; ++b)
                for (int w = 0; w < 2; ++w) {
                    V2Lay X = L;
                    std::swap(X.lane[lpos[a]], X.warp[w]);
                    std::swap(X.lane[lpos[b]], X.warp[1 - w]);
                    const int f = wf8(X);
                    if (f < best) {
                        best = f;
                        B = X;
                    }
                }
        L = B;
    };
    auto local_of = [](const V2Lay& L) {
        uint32_t m = 0;
        for (int t = 0; t < 4; ++t) m |= 1u << L.cfg[t];
        for (int t = 0; t < 2; ++t) m |= 1u << L.grp[t];
        return m;
    };
    auto unit = [](uint32_t b) -> uint16_t {
        const uint32_t L = 1u << b;
        return (uint16_t)((L ^ ((((L >> 4) ^ (L >> 7) ^ (L >> 10)) & 7u) << 1)) << 3);
    };
    std::vector<V2Lay> lay(count);
    std::vector<int> tr(count, 0);  // transition into gate i: 0 start (gather), 1 L, 2 X
    double cum = 1.0;
    for (int i = 0; i < count; ++i) {
        if (!(gd[i].k & kGateTC)) {
            cum = 1.0;
            continue;
        }
        const bool prev_tc = i > 0 && (gd[i - 1].k & kGateTC);
        int t = 0;
        if (prev_tc && cum * norms[i] <= 16.0) {
            const V2Lay& P = lay[i - 1];
            const uint32_t local = local_of(P) & ~(half_split ? (1u << P.grp[1]) : 0u);
            if ((lmask[i] & ~local) == 0) {
                t = 1;  // L: same rows, new roles of the 6 thread-local bits
                V2Lay& L = lay[i];
                order_cfg(i, -1, L.cfg);
                pair0(L);
                int g2[6], ng2 = 0;
                for (int b = 0; b < T; ++b)
                    if (((local & ~lmask[i]) >> b) & 1u) g2[ng2++] = b;
                L.grp[0] = g2[0];
                L.grp[1] = half_split ? P.grp[1] : g2[1];
                std::memcpy(L.lane, P.lane, sizeof L.lane);
                std::memcpy(L.warp, P.warp, sizeof L.warp);
            } else {
                // X: rows (c0, c1, L0, L1, L2 | warps); local = {L3, L4, c2, c3, j0, j1}
                const uint32_t lx = (1u << P.lane[3]) | (1u << P.lane[4]) | (1u << P.cfg[2]) | (1u << P.cfg[3]) |
                                    (1u << P.grp[0]) | (half_split ? 0u : (1u << P.grp[1]));
                if ((lmask[i] & ~lx) == 0 && ((lmask[i] >> P.lane[3]) & 1u)) {
                    t = 2;
                    V2Lay& L = lay[i];
                    order_cfg(i, P.lane[3], L.cfg);
                    int g2[6], ng2 = 0;
                    for (int b = 0; b < T; ++b)
                        if (((lx & ~lmask[i]) >> b) & 1u) g2[ng2++] = b;
                    L.grp[0] = g2[0];
                    L.grp[1] = half_split ? P.grp[1] : g2[1];
                    L.lane[0] = P.cfg[0];
                    L.lane[1] = P.cfg[1];
                    L.lane[2] = P.lane[0];
                    L.lane[3] = P.lane[1];
                    L.lane[4] = P.lane[2];
                    L.warp[0] = P.warp[0];
                    L.warp[1] = P.warp[1];
                }
            }
        }
        if (t == 0) {
            fresh(i, lay[i]);
            cum = 1.0;
        }
        cum *= norms[i];
        tr[i] = t;
    }
    // segments = maximal runs of gates joined by L / X transitions; the scale headroom
    // of a segment covers the product of its gates' norm bounds
    for (int i = 0; i < count; ++i) {
        if (!(gd[i].k & kGateTC)) continue;
        const V2Lay& L = lay[i];
        const bool start = tr[i] == 0;
        const bool end = i + 1 >= count || !(gd[i + 1].k & kGateTC) || tr[i + 1] == 0;
        int32_t k = (gd[i].k & ~(kGateRunStart | kGateRunEnd | kGateXNext | kGatePair0 | (0xff << kGateShiftBit))) | kGateV2;
        if (start) {
            double c = 1.0;
            for (int j = i; j < count && (gd[j].k & kGateTC) && (j == i || tr[j] != 0); ++j) c *= norms[j];
            const int shift = c > 1.0 ? std::min(100, (int)std::ceil(std::log2(c))) : 0;
            k |= kGateRunStart | (shift << kGateShiftBit);
        }
        if (end) k |= kGateRunEnd;
        if (!end && tr[i + 1] == 2) k |= kGateXNext;
        if (L.cfg[0] == 0) k |= kGatePair0;
        uint16_t u[20] = {0};
        for (int r = 0; r < 4; ++r) u[r] = unit((uint32_t)L.cfg[r]);
        for (int r = 0; r < 2; ++r) u[4 + r] = unit((uint32_t)L.grp[r]);
        for (int r = 0; r < 5; ++r) u[6 + r] = unit((uint32_t)L.lane[r]);
        for (int r = 0; r < 2; ++r) u[11 + r] = unit((uint32_t)L.warp[r]);
        if (!end) {
            const V2Lay& N = lay[i + 1];
            if (tr[i + 1] == 1) {
                // L: TMEM column (in this gate's D) of the next gate's roles cfg0..3, grp0..1
                const int roles[6] = {N.cfg[0], N.cfg[1], N.cfg[2], N.cfg[3], N.grp[0], N.grp[1]};
                for (int r = 0; r < 6; ++r) {
                    uint16_t v = 0;
                    for (int q = 0; q < 4; ++q)
                        if (L.cfg[q] == roles[r]) v = (uint16_t)(2u << q);
                    for (int q = 0; q < 2; ++q)
                        if (L.grp[q] == roles[r]) v = (uint16_t)(64u << q);
                    u[13 + r] = v;
                }
            } else {
                // X: 16x256b loads; the next gate's matrix bit 0 is this gate's lane bit 3
                // (load register pair), roles cfg1..3, grp0..1 -> TMEM address deltas of
                // lane bit 4 (lane + 16), config bits 2, 3 (columns 8, 16), groups (64, 128)
                const int roles[5] = {N.cfg[1], N.cfg[2], N.cfg[3], N.grp[0], N.grp[1]};
                for (int r = 0; r < 5; ++r) {
                    uint16_t v = 0;
                    if (roles[r] == L.lane[4]) v = 0x8000u;  // lane + 16 (the kernel expands it)
                    if (roles[r] == L.cfg[2]) v = 8;
                    if (roles[r] == L.cfg[3]) v = 16;
                    if (roles[r] == L.grp[0]) v = 64;
                    if (roles[r] == L.grp[1]) v = 128;
                    u[14 + r] = v;
                }
            }
        }
        gd[i].k = k;
        gd[i].mat_off = gd[i].mat_off;
        std::memcpy(v2_units(gd[i]), u, sizeof u);
        // matrix bit m <-> tile bit cfg[m]: constituent positions follow that order
        if (gate_fused[i] >= 0) {
            int asc[4];
            bits_of(lmask[i], asc);
            int rank_to_m[4];
            for (int a = 0; a < 4; ++a)
                for (int m = 0; m < 4; ++m)
                    if (L.cfg[m] == asc[a]) rank_to_m[a] = m;
            const FusedDesc& fd = fused[gate_fused[i]];
            for (int ci = fd.cons_begin; ci < fd.cons_begin + fd.cons_count; ++ci) {
                uint32_t pos = cons[ci].pos, np = pos;
                for (int j = 0; j < 4; ++j) {
                    const uint32_t pv = (pos >> (4 * j)) & 15u;
                    if (pv < 4) np = (np & ~(15u << (4 * j))) | ((uint32_t)rank_to_m[pv] << (4 * j));
                }
                cons[ci].pos = np;
            }
        }
    }
}

}  // namespace

qt_status plan_trajectory(const Plan& P, uint64_t seed, uint64_t traj, const ObsGroups& og,
                          TrajProgram& out, int mode) {
#ifdef QT_PLAN_PROFILE
    auto t_pp = std::chrono::steady_clock::now();
#endif
    // reset, keeping the vectors' capacity (callers reuse programs across batches)
    out.passes.clear();
    out.gates.clear();
    out.fused.clear();
    out.cons.clear();
    out.events.clear();
    out.records.clear();
    out.pool_size = 0;
    out.n_deferred = out.n_conventional = 0;
    out.alg_bytes = out.alg_flops = 0;
    const bool conventional = (mode == 1);  // no lower bounds, every channel reduces
    const int n = P.n;
    const int T = P.T;
    out.records.assign(P.n_recorded, -1);
    // ---- 1. draws + Alg. 2 first loop; build segments
    // per-thread scratch, reused across trajectories
    thread_local std::vector<std::vector<Item>> segs;
    thread_local size_t nsegs;
    nsegs = 1;
    if (segs.empty()) segs.emplace_back();
    segs[0].clear();
    auto new_seg = [&]() {
        if (segs.size() <= nsegs) segs.emplace_back();
        segs[nsegs++].clear();
    };
    struct Barrier { int event; uint64_t qmask; };
    thread_local std::vector<Barrier> barriers;
    barriers.clear();
    for (const PlanOp& op : P.ops) {
        if (op.kind == 0) {
            // sweep gates (P:262 parametrized circuits): variant = parameter set traj mod n_sets
            const int v = op.var_base + (op.n_kraus > 1 ? (int)(traj % (uint64_t)P.n_sets) : 0);
            if (!P.vars[v].identity) segs[nsegs - 1].push_back(Item{op.mask, v, -1, op.nq});
            continue;
        }
        const double u = draw(seed, (uint32_t)op.chan, kPurposeChannel, traj, 0);
        double r = u;
        int pick = -1;
        if (!conventional) {
            for (int i = 0; i < op.n_kraus; ++i) {
                if (r < op.pbar[i]) { pick = i; break; }
                r -= op.pbar[i];
            }
            if (pick < 0 && op.mixture) pick = op.n_kraus - 1;  // s == 1
        }
        if (pick >= 0) {
            ++out.n_deferred;
            if (op.record >= 0) out.records[op.record] = pick;
            const int v = op.var_base + pick;
            if (!P.vars[v].identity) segs[nsegs - 1].push_back(Item{op.mask, v, -1, op.nq});
            continue;
        }
        // conventional: barrier + device-chosen op opening the next segment
        ++out.n_conventional;
        EventDesc E;
        E.chan = op.chan;
        E.mat_off = 0;  // assigned below
        E.record = op.record;
        E.slot = 0;
        E.r = r;
        E.flags = conventional ? kEventNoBounds : 0;
        E.pad = 0;
        const int ev = (int)out.events.size();
        out.events.push_back(E);
        barriers.push_back(Barrier{ev, op.mask});
        new_seg();
        segs[nsegs - 1].push_back(Item{op.mask, -1, ev, op.nq});
    }
    QT_PP(0);
    // ---- 2.+3. fuse each segment, pack passes
    const uint64_t lowS = low_mask(std::min(P.CL, n));
    const uint64_t lowT = low_mask(T);
    int32_t pool = 0;
    thread_local std::vector<uint64_t> gate_masks;  // parallel to out.gates
    thread_local std::vector<double> gate_norms;    // parallel to out.gates: spectral-norm bound
    thread_local std::vector<int> gate_fused;       // parallel to out.gates: FusedDesc index or -1
    gate_masks.clear();
    gate_norms.clear();
    gate_fused.clear();
    auto alloc = [&](int d2) {
        const int32_t off = pool;
        pool += (d2 + 1) & ~1;  // keep 16-byte alignment
        return off;
    };
    for (size_t si = 0; si < nsegs; ++si) {
        const std::vector<Item>& items = segs[si];
        thread_local std::vector<FuseItem> fi;
        thread_local std::vector<int> fflat, foffs;
        fi.resize(items.size());
        for (size_t i = 0; i < items.size(); ++i) fi[i] = FuseItem{items[i].mask, items[i].var < 0};
        QT_PP(1);
        fuse_items(fi.data(), (int)fi.size(), P.f, fflat, foffs);
        QT_PP(2);
        thread_local std::vector<FusedGate> fg;
        fg.clear();
        for (size_t gi = 0; gi + 1 < foffs.size(); ++gi) {
            FusedGate x;
            x.items = fflat.data() + foffs[gi];
            x.n_items = foffs[gi + 1] - foffs[gi];
            x.mask = 0;
            x.special_event = -1;
            for (int it : x) x.mask |= items[it].mask;
            if (x.n_items == 1 && items[x.items[0]].var < 0) x.special_event = items[x.items[0]].event;
            if (x.special_event < 0)
                for (int it : x)
                    if (items[it].var < 0) return QT_EINVAL;  // fixed item fused (cannot happen)
            fg.push_back(x);
        }
        // pass packing
        thread_local std::vector<char> taken;
        taken.assign(fg.size(), 0);
        size_t remaining = fg.size();
        const bool last_seg = (si + 1 == nsegs);
        thread_local std::vector<size_t> seg_pass_idx;
        seg_pass_idx.clear();
        // tensor cores: a fused gate is padded to tc_k qubits with the lowest
        // qubits it does not touch, which must lie in the tile too
        auto padded = [&](const FusedGate& g) {
            uint64_t pm = g.mask;
            if (P.tc && g.special_event < 0)
                for (int q = 0; q < n && popc(pm) < P.tc_k; ++q) pm |= 1ull << q;
            return pm;
        };
        while (remaining > 0) {
            uint64_t S = lowS;
            uint64_t blocked = 0;
            thread_local std::vector<int> chosen;
            chosen.clear();
            for (size_t i = 0; i < fg.size(); ++i) {
                if (taken[i]) continue;
                const uint64_t gm = fg[i].mask;
                if (gm & blocked) { blocked |= gm; continue; }
                const uint64_t gp = padded(fg[i]);
                if (popc(S | gp) <= T && (!P.one_gate || chosen.empty()) &&
                    (int)chosen.size() < kMaxPassGates) {
                    S |= gp;
                    chosen.push_back((int)i);
                } else {
                    blocked |= gm;
                }
            }
            for (int i : chosen) taken[i] = 1;
            remaining -= chosen.size();
            PassDesc pd;
            pd.tile_mask = S;  // filled below
            pd.gate_begin = (int32_t)out.gates.size();
            pd.gate_count = (int32_t)chosen.size();
            pd.flags = kPassStore;
            pd.event = -1;
            pd.obs_begin = 0;
            pd.obs_count = 0;
            for (int i : chosen) {
                FusedGate& g = fg[i];
                GateDesc gd;
                std::memset(&gd, 0, sizeof gd);
                gd.k = popc(g.mask);
                gd.rpos = gd.tpos = 0;  // after S is final
                double gnorm = 1.0;
                for (int it : g)
                    if (items[it].var >= 0) gnorm *= P.vars[items[it].var].norm;
                if (g.special_event >= 0) {
                    const int d = 1 << gd.k;
                    gd.mat_off = alloc(d * d);
                    out.events[g.special_event].mat_off = gd.mat_off;
                } else {
                    // tensor cores: pad the fused gate to tc_k qubits (inside the tile)
                    const uint64_t pm = padded(g);
                    const int d = 1 << popc(pm);
                    // tensor cores: the GEMM operand, tc_gate_bytes(tc_k) bytes (complex64 units)
                    gd.mat_off = alloc((P.v2 || P.v3) ? kV2GateBytes / 8 : (P.tc ? tc_gate_bytes(P.tc_k) / 8 : d * d));
                    FusedDesc fd;
                    fd.mat_off = gd.mat_off;
                    fd.k = popc(pm) | (P.tc ? kGateTC : 0) | ((P.v2 || P.v3) ? kGateV2 : 0);
                    fd.cons_begin = (int32_t)out.cons.size();
                    fd.cons_count = (int32_t)g.n_items;
                    for (int it : g) {
                        ConsDesc c;
                        c.var = items[it].var;
                        uint32_t pos = 0;
                        int m = 0;
                        for (uint64_t mk = items[it].mask; mk; mk &= mk - 1, ++m) {
                            const int q = __builtin_ctzll(mk);
                            pos |= (uint32_t)popc(pm & low_mask(q)) << (4 * m);
                        }
                        c.pos = pos;
                        out.cons.push_back(c);
                    }
                    out.fused.push_back(fd);
                    if (P.tc) {
                        gd.k |= kGateTC;
                        g.mask = pm;  // layout over the padded qubit set
                    }
                }
                out.alg_flops += std::ldexp(1.0, n + (gd.k & 0xff) + 3);
                if (P.tc && (gd.k & kGateTC)) gd.k = P.tc_k | kGateTC;
                out.gates.push_back(gd);
                gate_masks.push_back(g.mask);
                gate_norms.push_back(gnorm);
                gate_fused.push_back(g.special_event >= 0 ? -1 : (int)out.fused.size() - 1);
            }
            seg_pass_idx.push_back(out.passes.size());
            out.passes.push_back(pd);
        }
        QT_PP(3);
        // barrier epilogue: rho_Q of the next conventional channel
        if (!last_seg) {
            const Barrier& b = barriers[si];
            if (seg_pass_idx.empty() || popc(out.passes[seg_pass_idx.back()].tile_mask | b.qmask) > T) {
                PassDesc pd;
                pd.tile_mask = lowS | b.qmask;
                pd.gate_begin = (int32_t)out.gates.size();
                pd.gate_count = 0;
                pd.flags = 0;
                pd.event = -1;
                pd.obs_begin = pd.obs_count = 0;
                seg_pass_idx.push_back(out.passes.size());
                out.passes.push_back(pd);
            }
            PassDesc& lp = out.passes[seg_pass_idx.back()];
            lp.tile_mask |= b.qmask;
            lp.flags |= kPassRho;
            lp.event = b.event;
        }
        // finalize tile masks, then tile-local gate positions
        for (size_t pi : seg_pass_idx) {
            PassDesc& pd = out.passes[pi];
            pd.tile_mask = fill_tile(pd.tile_mask, T, n);
            pd.rho_local = 0;
            pd.rho_nq = 0;
            pd.pad = 0;
            if (pd.flags & kPassRho) {
                const uint64_t qm = barriers[si].qmask;
                int i = 0;
                for (uint64_t mk = pd.tile_mask; mk; mk &= mk - 1, ++i)
                    if ((qm >> __builtin_ctzll(mk)) & 1u) pd.rho_local |= 1u << i;
                pd.rho_nq = popc(qm);
            }
            for (int g = 0; g < pd.gate_count; ++g) {
                GateDesc& gd = out.gates[pd.gate_begin + g];
                // 6-qubit tensor-core gates: every gate bit in registers (R = 6)
                const int R = (P.tc && P.tc_k == 6 && (gd.k & kGateTC)) ? 6 : P.R;
                gate_layout(gate_masks[pd.gate_begin + g], pd.tile_mask, T, R, gd.rpos, gd.tpos);
            }
            if (P.v2) {
                thread_local std::vector<uint32_t> lm;
                lm.resize(pd.gate_count);
                for (int g = 0; g < pd.gate_count; ++g) {
                    uint32_t l = 0;
                    int i = 0;
                    for (uint64_t mk = pd.tile_mask; mk; mk &= mk - 1, ++i)
                        if ((gate_masks[pd.gate_begin + g] >> __builtin_ctzll(mk)) & 1u) l |= 1u << i;
                    lm[g] = l;
                }
                v2_layouts(out.gates.data() + pd.gate_begin, lm.data(), gate_norms.data() + pd.gate_begin,
                           pd.gate_count, out.fused, out.cons, gate_fused.data() + pd.gate_begin);
            } else if (P.v3) {
                for (int g = 0; g < pd.gate_count; ++g) v3_lanes(out.gates[pd.gate_begin + g]);
            } else if (P.tc && P.tc_k == 4) {
                tc_runs(out.gates.data() + pd.gate_begin, gate_norms.data() + pd.gate_begin, pd.gate_count, T,
                        out.fused, out.cons, gate_fused.data() + pd.gate_begin);
                for (int g = 0; g < pd.gate_count; ++g)
                    if (out.gates[pd.gate_begin + g].k & kGateF16) out.fused[gate_fused[pd.gate_begin + g]].k |= kGateF16;
            }
        }
    }
    QT_PP(4);
    // ---- 4. final epilogue: block sums over the low T qubits (+ observables of
    // group 0), then read-only passes for the other observable groups
    if (og.final_pass) {
        const bool merge = !out.passes.empty() && out.passes.back().tile_mask == lowT &&
                           !(out.passes.back().flags & kPassRho);
        if (!merge) {
            PassDesc pd;
            pd.tile_mask = lowT;
            pd.gate_begin = (int32_t)out.gates.size();
            pd.gate_count = 0;
            pd.flags = 0;
            pd.event = -1;
            pd.obs_begin = pd.obs_count = 0;
            out.passes.push_back(pd);
        }
        PassDesc& fp = out.passes.back();
        fp.flags |= kPassFinal;
        if (!og.ranges.empty() && og.ranges[0].second > 0) {
            fp.flags |= kPassObs;
            fp.obs_begin = og.ranges[0].first;
            fp.obs_count = og.ranges[0].second;
        }
        for (size_t k = 1; k < og.ranges.size(); ++k) {
            PassDesc pd;
            pd.tile_mask = og.masks[k];
            pd.gate_begin = (int32_t)out.gates.size();
            pd.gate_count = 0;
            pd.flags = kPassObs;
            pd.event = -1;
            pd.obs_begin = og.ranges[k].first;
            pd.obs_count = og.ranges[k].second;
            out.passes.push_back(pd);
        }
    }
    for (auto& pd : out.passes) {  // tile bit i -> global qubit
        std::memset(pd.tq, 0, sizeof pd.tq);
        int i = 0;
        for (uint64_t mk = pd.tile_mask; mk; mk &= mk - 1) pd.tq[i++] = (uint8_t)__builtin_ctzll(mk);
        pd.slot = 0;
    }
    out.pool_size = pool;
    QT_PP(5);
    // algorithmic bytes: 2^(n+4) per storing pass, 2^(n+3) per read-only pass
    for (auto& pd : out.passes) out.alg_bytes += std::ldexp(1.0, n + ((pd.flags & kPassStore) ? 4 : 3));
    return QT_OK;
}

}  // namespace qt
