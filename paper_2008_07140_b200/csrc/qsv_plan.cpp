// Gate scheduler / fuser (see qsv_plan.h for the execution model).
//
// Dependency rule.  Gate B must stay after gate A when they share a qubit on
// which at least one of them acts non-diagonally; gates that act diagonally
// (in the computational basis) on every shared qubit commute.  Controls act
// diagonally on their qubit (gates.py:162-168 embeds controls as a
// block-diagonal), and so do all qubits of a diagonal gate - the same test the
// reference uses to route a gate to _k_diag/_k_scale (statevector.py:177).
//
// Greedy absorption in program order (both for passes over tile qubits and
// for stages over register qubits): a gate is taken when none of its qubits
// is blocked by an earlier deferred gate and its non-diagonal targets fit in
// the residency set (growing it up to capacity); otherwise it is deferred and
// blocks its qubits for the rest of the scan.  Taking gates in program order
// with this blocking rule keeps every emitted sequence a topological order of
// the dependency DAG.
#include "qsv_plan.h"

#include <algorithm>
#include <atomic>
#include <thread>
#include <bit>
#include <cstdlib>
#include <cstring>
#include <string>

namespace qsv {

static inline int popc(uint64_t x) { return std::popcount(x); }

void resolve_options(const qsv_options *opt, int n, int &m, int &r, int &L, int &s) {
    // L2 super-tiles are opt-in (super_qubits > tile_qubits): on B200 the
    // persistent super-pass kernel measured slower than flat passes for the
    // FP64-bound RQC/QFT workloads (grid-barrier tails), see DESIGN.md
    s = (opt && opt->super_qubits > 0) ? opt->super_qubits : 0;
    m = (opt && opt->tile_qubits > 0) ? opt->tile_qubits : 12;
    // 32 amplitudes per thread for the specialised kernels (measured best on
    // B200: fewer stages and barriers), 16 for the interpreted kernel
    const bool jit = opt ? (opt->jit > 0 || (opt->jit == 0 && n >= 16)) : n >= 16;
    r = (opt && opt->reg_qubits > 0) ? opt->reg_qubits : (jit ? 5 : 4);
    // forced low tile qubits: 3 keeps every warp access in full 128-byte lines
    // and frees tile slots for gates (C2 10 -> 8 passes, 67.3 -> 64.6 ms; QFT
    // 7 -> 5 passes, 47.8 -> 42.4 ms, with one CTA per tile); 5 was the
    // default while the pass kernels ran persistent grids
    L = (opt && opt->low_qubits > 0) ? opt->low_qubits : 3;
    m = std::min(std::min(m, kMaxTileQubits), n);
    r = std::max(std::min(std::min(r, kMaxRegQubits), m), std::min(2, m));
    m = std::min(m, r + 9);  // at most 512 threads per CTA (launch bound of pass_kernel)
    // leave room for a 2-target gate outside the forced low block
    L = std::max(0, std::min(L, m - 2));
}

int to_records(const qsv_gate *gates, int64_t n_gates, int n, std::vector<GateRec> &out, std::string &msg) {
    out.clear();
    out.reserve(n_gates);
    const uint64_t all = (n >= 64) ? ~0ull : ((1ull << n) - 1);
    for (int64_t i = 0; i < n_gates; ++i) {
        const qsv_gate &g = gates[i];
        GateRec r;
        r.nt = g.n_targets;
        if (r.nt < 1 || r.nt > 2) {
            msg = "gate " + std::to_string(i) + ": " + std::to_string(g.n_targets) + " targets (only 1 or 2)";
            return QSV_E_UNSUPPORTED;
        }
        uint64_t tmask = 0;
        for (int k = 0; k < r.nt; ++k) {
            r.t[k] = g.targets[k];
            if (r.t[k] < 0 || r.t[k] >= n) {
                msg = "gate " + std::to_string(i) + ": target qubit " + std::to_string(r.t[k]) + " out of range";
                return QSV_E_PARSE;
            }
            tmask |= 1ull << r.t[k];
        }
        if (r.nt == 2 && r.t[0] == r.t[1]) {
            msg = "gate " + std::to_string(i) + ": repeated target";
            return QSV_E_PARSE;
        }
        r.cmask = g.control_mask;
        if ((r.cmask & ~all) || (r.cmask & tmask)) {
            msg = "gate " + std::to_string(i) + ": control mask out of range or overlapping a target";
            return QSV_E_PARSE;
        }
        const int d = 1 << r.nt;
        bool diag = true;
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) {
                r.u[a * d + b] = cd(g.u[2 * (a * d + b)], g.u[2 * (a * d + b) + 1]);
                if (a != b && r.u[a * d + b] != cd(0.0, 0.0)) diag = false;
            }
        r.diag = diag;
        r.nmask = diag ? 0 : tmask;
        r.dmask = r.cmask | (diag ? tmask : 0);
        out.push_back(r);
    }
    return QSV_OK;
}

namespace {

// Rough FP64 work per amplitude of one gate in a specialised pass (cost
// model for balancing passes): a non-diagonal 1-qubit gate is 2-4 FP64
// operations per amplitude after coefficient absorption, a dense 2-qubit gate
// ~8, diagonals are mostly absorbed.
inline double gate_work(const GateRec &g) {
    if (g.diag) return 0.25;
    return g.nt == 1 ? 3.0 : 8.0;
}

struct Absorber {
    uint64_t resident = 0;  // qubits currently resident (tile or registers)
    int capacity = 0;
    uint64_t blockN = 0, blockD = 0;
    double budget = 0, work = 0;  // optional cap on the summed gate_work (0: none)

    // true when gate g is taken
    bool offer(const GateRec &g) {
        const uint64_t touched = g.nmask | g.dmask;
        bool blocked = (touched & blockN) || (g.nmask & blockD);
        if (!blocked && budget > 0 && work + gate_work(g) > budget) blocked = true;
        if (!blocked) {
            const uint64_t need = g.nmask & ~resident;
            if (popc(resident | need) <= capacity) {
                resident |= need;
                work += gate_work(g);
                return true;
            }
        }
        blockN |= g.nmask;
        blockD |= g.dmask;
        return false;
    }
};

// Local bit index of global qubit q inside the tile (tile_mask sorted ascending).
inline int local_bit(uint64_t tile_mask, int q) {
    if (!((tile_mask >> q) & 1)) return -1;
    return popc(tile_mask & ((1ull << q) - 1));
}

inline uint64_t deposit(uint64_t v, uint64_t mask) {
    uint64_t out = 0;
    for (int bit = 0; mask; ++bit) {
        const uint64_t low = mask & (~mask + 1);
        if ((v >> bit) & 1) out |= low;
        mask ^= low;
    }
    return out;
}

using StageOp = GlobalOp;

inline uint64_t op_nmask(const StageOp &o) {
    if (o.kind == QSV_OP_MAT1) return 1ull << o.qa;
    if (o.kind == QSV_OP_MAT2) return (1ull << o.qa) | (1ull << o.qb);
    return 0;
}
inline uint64_t op_dmask(const StageOp &o) {
    uint64_t d = o.cmask;
    if (o.kind == QSV_OP_DIAG1) d |= 1ull << o.qa;
    if (o.kind == QSV_OP_DIAG2) d |= (1ull << o.qa) | (1ull << o.qb);
    return d;
}

StageOp make_op(const GateRec &g) {
    StageOp o;
    o.cmask = g.cmask;
    o.qa = g.t[0];
    o.qb = g.nt == 2 ? g.t[1] : -1;
    if (g.nt == 1) {
        o.kind = g.diag ? QSV_OP_DIAG1 : QSV_OP_MAT1;
        if (g.diag) {
            o.m[0] = g.u[0];
            o.m[1] = g.u[3];
        } else {
            for (int k = 0; k < 4; ++k) o.m[k] = g.u[k];
        }
    } else {
        o.kind = g.diag ? QSV_OP_DIAG2 : QSV_OP_MAT2;
        if (g.diag) {
            for (int k = 0; k < 4; ++k) o.m[k] = g.u[5 * k];
        } else {
            for (int k = 0; k < 16; ++k) o.m[k] = g.u[k];
        }
    }
    return o;
}

// 2x2 products for the single-qubit peephole: returns new = b * a (apply a, then b).
void mul2(const cd *b, const cd *a, cd *out) {
    cd r[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) r[2 * i + j] = b[2 * i] * a[j] + b[2 * i + 1] * a[2 + j];
    for (int k = 0; k < 4; ++k) out[k] = r[k];
}

// Appends `o` to the stage, merging it into an earlier single-qubit op of the
// same kind (MAT1 with MAT1, DIAG1 with DIAG1) on the same target with the same
// controls when every op in between commutes with it.  A diagonal is not folded
// into a dense 2x2: the kernel applies a phase to half the amplitudes for 2
// FP64 ops per amplitude, while a fused complex 2x2 costs 8 against 4 for the
// real / RX-like 2x2 it would replace.
void append_fused(std::vector<StageOp> &ops, const StageOp &o) {
    if (o.kind == QSV_OP_MAT1 || o.kind == QSV_OP_DIAG1) {
        const uint64_t q = 1ull << o.qa;
        const bool o_diag = o.kind == QSV_OP_DIAG1;
        for (int k = (int)ops.size() - 1; k >= 0; --k) {
            StageOp &p = ops[k];
            if (p.kind == o.kind && p.qa == o.qa && p.cmask == o.cmask) {
                if (o_diag) {
                    p.m[0] = o.m[0] * p.m[0];
                    p.m[1] = o.m[1] * p.m[1];
                } else {
                    cd r[4];
                    mul2(o.m, p.m, r);
                    for (int i = 0; i < 4; ++i) p.m[i] = r[i];
                }
                return;
            }
            // can o move before p?  every shared qubit must be diagonal for both
            const uint64_t pn = op_nmask(p), pd = op_dmask(p);
            const uint64_t on = o_diag ? 0 : q, od = o.cmask | (o_diag ? q : 0);
            const uint64_t shared = (pn | pd) & (on | od);
            if (shared & (pn | on)) break;
        }
    }
    ops.push_back(o);
}

inline bool is_zero(cd z) { return z.real() == 0.0 && z.imag() == 0.0; }

int mat1_variant(const cd *u) {
    bool real = true;
    for (int i = 0; i < 4; ++i) real &= u[i].imag() == 0.0;
    if (real) return V_REAL;
    if (u[0].imag() == 0.0 && u[3].imag() == 0.0 && u[1].real() == 0.0 && u[2].real() == 0.0) return V_RXL;
    return V_GEN;
}

inline int factor_mode(cd f) {
    if (f == cd(1.0, 0.0)) return 0;
    if (f == cd(-1.0, 0.0)) return 1;
    return 2;
}

// Lowers one global op to the device record for a stage whose register
// positions are given by `regpos_of_local` inside tile `tmask`.
DevOp lower_op(const StageOp &o, int n, uint64_t tmask, const int32_t *regpos_of_local) {
    DevOp d;
    std::memset(&d, 0, sizeof(d));
    // qubit class: register position (>= 0) or scalar descriptor
    auto reg_of = [&](int q) -> int {
        const int lb = local_bit(tmask, q);
        return lb >= 0 ? regpos_of_local[lb] : -1;
    };
    auto scalar_of = [&](int q) -> uint32_t {
        const int lb = local_bit(tmask, q);
        return lb < 0 ? (uint32_t)(kScalarExt + q) : (uint32_t)lb;
    };
    uint32_t kind = 0, var = 0, a = kNoReg, b = kNoReg, modes = 0, src = 0;
    uint32_t sa = kNoScalar, sb = kNoScalar;
    uint64_t cmask = o.cmask;
    cd f[4];
    if (o.kind == QSV_OP_DIAG1 || o.kind == QSV_OP_DIAG2) {
        kind = K_DIAG;
        int qa = -1, qb;
        if (o.kind == QSV_OP_DIAG1) {
            // a controlled 1-qubit diagonal is a 2-qubit diagonal over (control, target):
            // d = [1, 1, d0, d1]; prefer a register-resident control so the
            // class selection is compile-time in the kernel
            qb = o.qa;
            f[0] = o.m[0];
            f[1] = o.m[1];
            f[2] = f[3] = cd(1.0, 0.0);
            int best = -1, best_rank = 9;
            for (int q = 0; q < n; ++q) {
                if (!((cmask >> q) & 1)) continue;
                const int rank = reg_of(q) >= 0 ? 0 : (local_bit(tmask, q) >= 0 ? 1 : 2);
                if (rank < best_rank) {
                    best_rank = rank;
                    best = q;
                }
            }
            if (best >= 0) {
                qa = best;
                cmask &= ~(1ull << best);
                f[2] = o.m[0];
                f[3] = o.m[1];
                f[0] = f[1] = cd(1.0, 0.0);
            }
        } else {
            qa = o.qa;
            qb = o.qb;
            for (int i = 0; i < 4; ++i) f[i] = o.m[i];
        }
        if (qa >= 0) {
            const int ra = reg_of(qa);
            if (ra >= 0) a = (uint32_t)ra;
            else sa = scalar_of(qa);
        }
        const int rb = reg_of(qb);
        if (rb >= 0) b = (uint32_t)rb;
        else sb = scalar_of(qb);
        var = (a != kNoReg ? D_A : 0) | (b != kNoReg ? D_B : 0);
        for (int i = 0; i < 4; ++i) {
            modes |= (uint32_t)factor_mode(f[i]) << (2 * i);
            d.m[2 * i] = f[i].real();
            d.m[2 * i + 1] = f[i].imag();
        }
    } else if (o.kind == QSV_OP_MAT1) {
        kind = K_MAT1;
        a = (uint32_t)reg_of(o.qa);
        var = mat1_variant(o.m);
        for (int i = 0; i < 4; ++i) {
            d.m[2 * i] = o.m[i].real();
            d.m[2 * i + 1] = o.m[i].imag();
        }
    } else {
        kind = K_MAT2;
        a = (uint32_t)reg_of(o.qa);
        b = (uint32_t)reg_of(o.qb);
        bool perm = true;
        int srcs[4] = {0, 0, 0, 0};
        for (int r = 0; r < 4 && perm; ++r) {
            int nz = 0;
            for (int c = 0; c < 4; ++c)
                if (!is_zero(o.m[4 * r + c])) {
                    ++nz;
                    srcs[r] = c;
                }
            perm = nz == 1;
        }
        if (perm) {
            var = V_PERM;
            for (int r = 0; r < 4; ++r) {
                src |= (uint32_t)srcs[r] << (2 * r);
                const cd ph = o.m[4 * r + srcs[r]];
                modes |= (uint32_t)factor_mode(ph) << (2 * r);
                d.m[2 * r] = ph.real();
                d.m[2 * r + 1] = ph.imag();
            }
        } else {
            var = V_GEN;
            for (int i = 0; i < 16; ++i) {
                d.m[2 * i] = o.m[i].real();
                d.m[2 * i + 1] = o.m[i].imag();
            }
        }
    }
    uint32_t rc = 0, tc = 0;
    uint64_t ec = 0;
    for (int q = 0; q < n; ++q) {
        if (!((cmask >> q) & 1)) continue;
        const int rq = reg_of(q);
        const int lb = local_bit(tmask, q);
        if (rq >= 0) rc |= 1u << rq;
        else if (lb >= 0) tc |= 1u << lb;
        else ec |= 1ull << q;
    }
    d.code = kind | var << 4 | a << 8 | b << 12 | modes << 16 | src << 24;
    d.rs = rc | sa << 8 | sb << 16;
    d.tc = tc;
    d.ec = ec;
    return d;
}

}  // namespace

namespace {

inline uint64_t padded_tile(uint64_t res, uint64_t pool, int n, int m) {
    for (int q = 0; q < n && popc(res) < m; ++q)
        if ((pool >> q) & 1) res |= 1ull << q;
    return res;
}

inline bool conflict(const GateRec &a, const GateRec &b) {
    return (a.nmask & (b.nmask | b.dmask)) || (b.nmask & (a.nmask | a.dmask));
}

// Program-order scan with a FIXED tile: a gate is taken when its non-diagonal
// targets lie in the tile and no earlier deferred gate blocks it.  Returns the
// number taken.
int scan_fixed_tile(const std::vector<GateRec> &recs, const std::vector<int> &rem, uint64_t tile,
                    std::vector<int> *taken = nullptr, std::vector<int> *deferred = nullptr) {
    uint64_t bN = 0, bD = 0;
    int count = 0;
    for (int gi : rem) {
        const GateRec &g = recs[gi];
        if (!(((g.nmask | g.dmask) & bN) || (g.nmask & bD)) && !(g.nmask & ~tile)) {
            ++count;
            if (taken) taken->push_back(gi);
            continue;
        }
        bN |= g.nmask;
        bD |= g.dmask;
        if (deferred) deferred->push_back(gi);
    }
    return count;
}

// The greedy absorber fixes the tile by first come, first served.  Local
// search over single-qubit swaps (keeping the forced low qubits) then picks
// the tile that absorbs the most gates of the remaining stream, which cuts
// the number of HBM passes (C2, m = 12: 13 -> 10 passes).  QSV_TILE_SEARCH=0
// restores the plain greedy tiles.
uint64_t search_tile(const std::vector<GateRec> &recs, const std::vector<int> &rem, uint64_t tile, uint64_t fixed,
                     int n, uint64_t universe = ~0ull) {
    int best = scan_fixed_tile(recs, rem, tile);
    for (bool improved = true; improved;) {
        improved = false;
        for (int a = 0; a < n && !improved; ++a) {
            if (!((tile >> a) & 1) || ((fixed >> a) & 1)) continue;
            for (int b = 0; b < n && !improved; ++b) {
                if (((tile >> b) & 1) || !((universe >> b) & 1)) continue;
                const uint64_t t2 = tile ^ (1ull << a) ^ (1ull << b);
                const int c = scan_fixed_tile(recs, rem, t2);
                if (c > best) {
                    best = c;
                    tile = t2;
                    improved = true;
                }
            }
        }
    }
    return tile;
}

// Number of passes the greedy planner (absorb + single-swap search) needs for
// `rem` (rollout for the look-ahead tile choice below); stops at `cap`.
int rollout_passes(const std::vector<GateRec> &recs, std::vector<int> cur, uint64_t low, uint64_t all, int n, int m,
                   int cap) {
    int passes = 0;
    while (!cur.empty() && passes < cap) {
        Absorber tile;
        tile.resident = low;
        tile.capacity = m;
        for (int gi : cur) tile.offer(recs[gi]);
        const uint64_t res = search_tile(recs, cur, padded_tile(tile.resident, all, n, m), low, n);
        std::vector<int> t, d;
        scan_fixed_tile(recs, cur, res, &t, &d);
        cur.swap(d);
        ++passes;
    }
    return cur.empty() ? passes : cap + 1;
}

// Modeled time of one pass in FP64-instructions-per-amplitude units: a pass costs
// max(HBM floor, FP64 work); the floor (~65 FP64/amp on B200: 32 B/amp at ~6.9 TB/s
// vs ~78 % of the DFMA rate) and the work (gate_work ~ 1.5 units per FP64/amp).
double modeled_pass_time(const std::vector<GateRec> &recs, const std::vector<int> &taken) {
    double w = 0;
    for (int gi : taken) w += gate_work(recs[gi]);
    return std::max(65.0, w / 1.5);
}

// The look-ahead minimises the summed modeled pass time of the completion rather than the
// number of passes: heavy front passes + light tail passes cost more than balanced ones of
// the same count (a pass costs ~max(HBM time, FP64 time)).  Measured on B200, three
// interleaved rounds: C2 52.7 -> 51.0 ms (the same 7 passes and 579 FP64/amp, spread
// 115/95/66/96/90/73/45 instead of 118/104/85/115/91/50/16), n = 32 229.9 -> 227.3 ms, QFT
// unchanged (same plan).  A model with a per-stage term fitted to per-pass times (0.7 ms per
// stage) chose worse plans (C2 51.9 ms, n = 32 8 passes 244 ms): the crude model stays.
// qsv_options.plan_objective = 1 (or QSV_PLAN_OBJECTIVE=passes) restores the pass-count
// objective: C5's Pauli-carrying trajectories run faster on front-loaded plans (1024
// trajectories 0.79 s vs 1.06-1.20 s on time-balanced plans).
thread_local int t_plan_objective = 0;
bool objective_time() {
    static const int env = [] {
        const char *e = std::getenv("QSV_PLAN_OBJECTIVE");
        return !e ? 0 : std::string(e) == "passes" ? 1 : std::string(e) == "time" ? 2 : 0;
    }();
    const int o = env ? env : t_plan_objective;
    return o != 1;
}

// Summed modeled time of the greedy completion of `cur` (stops above `cap`).
double rollout_time(const std::vector<GateRec> &recs, std::vector<int> cur, uint64_t low, uint64_t all, int n, int m,
                    double cap) {
    double t = 0;
    while (!cur.empty() && t <= cap) {
        Absorber tile;
        tile.resident = low;
        tile.capacity = m;
        for (int gi : cur) tile.offer(recs[gi]);
        const uint64_t res = search_tile(recs, cur, padded_tile(tile.resident, all, n, m), low, n);
        std::vector<int> tk, d;
        scan_fixed_tile(recs, cur, res, &tk, &d);
        t += modeled_pass_time(recs, tk);
        cur.swap(d);
    }
    return cur.empty() ? t : cap + 1.0;
}

// Look-ahead tile choice (QSV_PLAN_ROLLOUT=K): among the best tile and its
// single-swap neighbours absorbing at least 70 % as many gates, the K with the
// most gates are completed greedily; the tile whose completion needs the fewest
// passes wins (ties: more gates now).  Minimises HBM passes rather than
// maximising each pass.
uint64_t lookahead_tile(const std::vector<GateRec> &recs, const std::vector<int> &rem, uint64_t best, uint64_t fixed,
                        uint64_t all, int n, int m, int K) {
    const int best_count = scan_fixed_tile(recs, rem, best);
    std::vector<std::pair<int, uint64_t>> cands{{best_count, best}};
    for (int a = 0; a < n; ++a) {
        if (!((best >> a) & 1) || ((fixed >> a) & 1)) continue;
        for (int b = 0; b < n; ++b) {
            if ((best >> b) & 1) continue;
            const uint64_t t2 = best ^ (1ull << a) ^ (1ull << b);
            const int c = scan_fixed_tile(recs, rem, t2);
            const int thr = std::getenv("QSV_PLAN_ROLLOUT_PCT") ? std::atoi(std::getenv("QSV_PLAN_ROLLOUT_PCT")) : 70;
            if (c * 100 >= best_count * thr) cands.push_back({c, t2});
        }
    }
    std::stable_sort(cands.begin() + 1, cands.end(), [](auto &x, auto &y) { return x.first > y.first; });
    if ((int)cands.size() > K) cands.resize(K);
    // the rollouts are independent: run them on up to 16 host threads, each capped
    // by the best completion found so far (a capped rollout returns cap + 1, which
    // never wins), then pick in candidate order - the same choice as a serial scan
    std::vector<int> passes(cands.size(), 1 << 30);
    std::atomic<int> best_so_far{1 << 30};
    std::atomic<size_t> next{0};
    const bool by_time = objective_time();
    auto work = [&] {
        for (size_t k; (k = next.fetch_add(1)) < cands.size();) {
            std::vector<int> t, d;
            scan_fixed_tile(recs, rem, cands[k].second, &t, &d);
            int p;
            if (by_time) {
                // modeled time in 1/16 units (ints keep the atomic pruning bound)
                const double now = modeled_pass_time(recs, t);
                const double rest = rollout_time(recs, d, fixed, all, n, m, best_so_far.load() / 16.0 - now);
                p = (int)std::min(1e9, 16.0 * (now + rest));
            } else {
                p = rollout_passes(recs, d, fixed, all, n, m, best_so_far.load());
            }
            passes[k] = p;
            for (int cur = best_so_far.load(); p < cur && !best_so_far.compare_exchange_weak(cur, p);) {
            }
        }
    };
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t nt = std::min<size_t>(hw, cands.size());
    if (nt <= 1) {
        work();
    } else {
        std::vector<std::thread> pool;
        for (size_t t = 0; t < nt; ++t) pool.emplace_back(work);
        for (auto &th : pool) th.join();
    }
    uint64_t choice = best;
    int best_passes = 1 << 30, choice_count = -1;
    for (size_t k = 0; k < cands.size(); ++k) {
        const int p = passes[k];
        if (p < best_passes || (p == best_passes && cands[k].first > choice_count)) {
            best_passes = p;
            choice = cands[k].second;
            choice_count = cands[k].first;
        }
    }
    return choice;
}

// Greedy absorption front-loads the FP64 work: the first passes take every
// gate they can and run compute-bound while the last ones are HBM-bound.  A
// pass costs ~max(HBM time, FP64 time), so gates at the tail of a heavy pass
// are pushed into the next pass when that lowers the summed cost: a gate may
// move when its non-diagonal targets lie in the next pass's tile and no later
// gate of its own pass depends on it; it becomes the first gate of the next
// pass (everything there that conflicts with it was blocked behind it).  The
// threshold (QSV_BALANCE_WORK, gate_work units) is the work at which a pass
// turns compute-bound.  Opt-in: on C2 the receiving passes slowed down far more
// than the FP64 model predicts (extra stages / runtime factors), net +2-5 ms.
void balance_passes(const std::vector<GateRec> &recs, std::vector<std::vector<int>> &gates,
                    const std::vector<uint64_t> &res, uint64_t pool, int n, int m) {
    const char *env = std::getenv("QSV_BALANCE_WORK");
    const double H = env ? std::atof(env) : 0.0;
    if (H <= 0 || gates.size() < 2) return;
    std::vector<double> w(gates.size(), 0.0);
    for (size_t k = 0; k < gates.size(); ++k)
        for (int gi : gates[k]) w[k] += gate_work(recs[gi]);
    auto cost = [&](double a, double b) { return std::max(H, a) + std::max(H, b); };
    for (int sweep = 0; sweep < 8; ++sweep) {
        bool moved = false;
        for (size_t k = gates.size() - 1; k-- > 0;) {
            const uint64_t next_tile = padded_tile(res[k + 1], pool, n, m);
            std::vector<int> &cur = gates[k];
            std::vector<int> moving;  // program order is restored below
            uint64_t later_n = 0, later_d = 0;  // qubits of the gates staying after position j
            for (size_t j = cur.size(); j-- > 0;) {
                const GateRec &g = recs[cur[j]];
                const double gw = gate_work(g);
                const bool free_of_later = !((g.nmask | g.dmask) & later_n) && !(g.nmask & later_d);
                if (free_of_later && !(g.nmask & ~next_tile) && cost(w[k] - gw, w[k + 1] + gw) < cost(w[k], w[k + 1]) - 1e-9) {
                    w[k] -= gw;
                    w[k + 1] += gw;
                    moving.push_back(cur[j]);
                    cur.erase(cur.begin() + (long)j);
                    moved = true;
                } else {
                    later_n |= g.nmask;
                    later_d |= g.dmask;
                }
            }
            if (!moving.empty()) {
                std::reverse(moving.begin(), moving.end());
                gates[k + 1].insert(gates[k + 1].begin(), moving.begin(), moving.end());
            }
        }
        if (!moved) break;
    }
}

// Emits one pass (tile + register stages) for `taken` (program order) into P.
// The tile holds the forced low qubits plus the non-diagonal targets of
// `taken`, padded with the lowest qubits of `pool` (the super-tile).
void emit_pass(Plan &P, const std::vector<GateRec> &recs, const std::vector<int> &taken, uint64_t tile_res,
               uint64_t pool, int r_pass = 0) {
    const int n = P.n, m = P.m, r = r_pass > 0 ? r_pass : P.r;
    uint64_t tmask = tile_res;
    for (int q = 0; q < n && popc(tmask) < m; ++q)
        if ((pool >> q) & 1) tmask |= 1ull << q;

    DevPass dp;
    std::memset(&dp, 0, sizeof(dp));
    dp.tile_mask = tmask;
    dp.m = m;
    dp.r = r;
    {
        int j = 0;
        for (int q = 0; q < n; ++q)
            if ((tmask >> q) & 1) dp.tq[j++] = q;
    }
    for (int e = 0; e < (1 << kLoTabBits); ++e) dp.lo_tab[e] = (e < (1 << m)) ? deposit(e, tmask) : 0;
    for (int e = 0; e < (1 << kHiTabBits); ++e)
        dp.hi_tab[e] = (m > kLoTabBits && e < (1 << (m - kLoTabBits))) ? deposit((uint64_t)e << kLoTabBits, tmask) : 0;
    dp.stage_begin = (int32_t)P.stages.size();
    P.pass_op_begin.push_back((int64_t)P.ops.size());

    // stages over register qubits
    std::vector<int> rem = taken;
    int stage_in_pass = 0;
    while (!rem.empty()) {
        Absorber regs;
        regs.capacity = r;
        std::vector<int> st_taken, st_def;
        for (int gi : rem) (regs.offer(recs[gi]) ? st_taken : st_def).push_back(gi);
        uint64_t rmask = regs.resident;
        // pad with the highest unused tile qubits
        for (int q = n - 1; q >= 0 && popc(rmask) < r; --q)
            if (((tmask >> q) & 1) && !((rmask >> q) & 1)) rmask |= 1ull << q;
        // the same local search as for tiles, over the pass's tile qubits
        // (C2: 27 -> 25 stages, 73.2 -> 71.4 ms; QSV_STAGE_SEARCH=0 disables)
        static const bool stage_search = !std::getenv("QSV_STAGE_SEARCH") || std::atoi(std::getenv("QSV_STAGE_SEARCH")) != 0;
        if (stage_search && !st_def.empty()) {
            rmask = search_tile(recs, rem, rmask, 0, n, tmask);
            st_taken.clear();
            st_def.clear();
            scan_fixed_tile(recs, rem, rmask, &st_taken, &st_def);
        }

        std::vector<StageOp> sops;
        for (int gi : st_taken) append_fused(sops, make_op(recs[gi]));

        DevStage ds;
        std::memset(&ds, 0, sizeof(ds));
        int k = 0;
        int32_t regpos_of_local[64];
        for (int j = 0; j < 64; ++j) regpos_of_local[j] = -1;
        for (int q = 0; q < n; ++q) {
            if ((rmask >> q) & 1) {
                const int lb = local_bit(tmask, q);
                ds.rb[k] = lb;
                regpos_of_local[lb] = k;
                ds.reg_local_mask |= 1u << lb;
                ++k;
            }
        }
        ds.op_begin = (int32_t)P.ops.size();
        for (const StageOp &o : sops) {
            P.ops.push_back(lower_op(o, n, tmask, regpos_of_local));
            P.gops.push_back(o);
            P.op_stage.push_back(stage_in_pass);
        }
        ds.op_end = (int32_t)P.ops.size();
        P.stages.push_back(ds);
        P.stage_regs.push_back(rmask);
        ++stage_in_pass;
        rem.swap(st_def);
    }
    dp.stage_end = (int32_t)P.stages.size();
    P.passes.push_back(dp);
}

}  // namespace

namespace {

bool is_plain_swap(const GateRec &g) {
    if (g.nt != 2 || g.cmask) return false;
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            const bool one = (a == 0 && b == 0) || (a == 3 && b == 3) || (a == 1 && b == 2) || (a == 2 && b == 1);
            if (g.u[a * 4 + b] != cd(one ? 1.0 : 0.0, 0.0)) return false;
        }
    return true;
}

GateRec swap_rec(int a, int b) {
    GateRec g;
    g.nt = 2;
    g.t[0] = a;
    g.t[1] = b;
    for (int k = 0; k < 16; ++k) g.u[k] = 0;
    g.u[0] = g.u[6] = g.u[9] = g.u[15] = 1;
    g.nmask = (1ull << a) | (1ull << b);
    return g;
}

}  // namespace

// SWAP gates (uncontrolled) move no data here: they permute the map from
// logical to physical qubits and every later gate is renamed through it
// (QFT's bit-reversal SWAP layers, C4, disappear entirely: the forward and
// the inverse layer cancel).  If the final map is not the identity, explicit
// SWAPs on physical qubits restore the order at the end.
std::vector<GateRec> relabel_swaps(const std::vector<GateRec> &in, int n) {
    bool any = false;
    for (const GateRec &g : in) any |= is_plain_swap(g);
    if (!any || (std::getenv("QSV_RELABEL_SWAPS") && std::atoi(std::getenv("QSV_RELABEL_SWAPS")) == 0)) return in;
    std::vector<int> phys(n);  // logical -> physical
    for (int q = 0; q < n; ++q) phys[q] = q;
    auto remap = [&](uint64_t mask) {
        uint64_t out = 0;
        for (int q = 0; q < n; ++q)
            if ((mask >> q) & 1) out |= 1ull << phys[q];
        return out;
    };
    std::vector<GateRec> out;
    out.reserve(in.size());
    for (const GateRec &g : in) {
        if (is_plain_swap(g)) {
            std::swap(phys[g.t[0]], phys[g.t[1]]);
            continue;
        }
        GateRec h = g;
        for (int k = 0; k < g.nt; ++k) h.t[k] = phys[g.t[k]];
        h.cmask = remap(g.cmask);
        h.nmask = remap(g.nmask);
        h.dmask = remap(g.dmask);
        out.push_back(h);
    }
    // restore: logical a back to physical a
    for (int a = 0; a < n; ++a) {
        if (phys[a] == a) continue;
        int b = 0;
        while (phys[b] != a) ++b;  // logical b currently sits on physical a
        out.push_back(swap_rec(phys[a], a));
        phys[b] = phys[a];
        phys[a] = a;
    }
    return out;
}

// Distributed layout (distributed.py).  With the state sharded
// over 2^g ranks only n - g qubits are local; a gate may act non-diagonally
// only on local qubits.  The stream is cut into SEGMENTS, each run with one
// fixed LOCAL SET of `capacity` logical qubits; between segments the qubits
// leaving / entering the local set are exchanged (one all-to-all).  Each
// segment takes every remaining gate its local set admits under the same
// dependency/blocking rule as the pass planner; the set itself starts from the
// previous one with the first blocked gate's targets brought in (evicting the
// local qubits whose next non-diagonal use is furthest away, Belady), then the
// single-swap local search maximises the gates absorbed.  With `free_initial`
// (the state is a basis state, layout-free) the first set is chosen freely.
int plan_segments(const std::vector<GateRec> &recs, int n, int capacity, uint64_t init_local, bool free_initial,
                  std::vector<int32_t> &gate_seg, std::vector<uint64_t> &seg_local) {
    const uint64_t all = n >= 64 ? ~0ull : ((1ull << n) - 1);
    gate_seg.assign(recs.size(), -1);
    seg_local.clear();
    std::vector<int> rem(recs.size());
    for (size_t i = 0; i < recs.size(); ++i) rem[i] = (int)i;
    uint64_t local = init_local & all;
    if (popc(local) != capacity) return QSV_E_PARSE;
    bool first = true;
    while (!rem.empty()) {
        uint64_t cand = local;
        if (first && free_initial) {
            Absorber a;
            a.capacity = capacity;
            for (int gi : rem) a.offer(recs[gi]);
            cand = padded_tile(a.resident, all, n, capacity);
        }
        first = false;
        // next non-diagonal use of every qubit (position in rem)
        std::vector<size_t> next(n, rem.size());
        for (size_t k = rem.size(); k-- > 0;)
            for (int q = 0; q < n; ++q)
                if ((recs[rem[k]].nmask >> q) & 1) next[q] = k;
        const GateRec &g0 = recs[rem[0]];
        uint64_t need = g0.nmask & ~cand;
        while (need) {
            int victim = -1;
            for (int q = 0; q < n; ++q)
                if (((cand >> q) & 1) && !((g0.nmask >> q) & 1) && (victim < 0 || next[q] > next[victim])) victim = q;
            const uint64_t in = need & (~need + 1);
            cand = (cand & ~(1ull << victim)) | in;
            need ^= in;
        }
        cand = search_tile(recs, rem, cand, 0, n, all);
        std::vector<int> taken, deferred;
        scan_fixed_tile(recs, rem, cand, &taken, &deferred);
        if (taken.empty()) return QSV_E_UNSUPPORTED;  // unreachable: rem[0] always fits
        for (int gi : taken) gate_seg[gi] = (int32_t)seg_local.size();
        seg_local.push_back(cand);
        local = cand;
        rem.swap(deferred);
    }
    return QSV_OK;
}

Plan build_single_pass(const std::vector<GateRec> &recs, const std::vector<int32_t> &taken, uint64_t tile_mask, int n,
                       int m, int r, int L) {
    Plan Q;
    Q.recs = recs;
    Q.n = n;
    Q.m = m;
    Q.r = r;
    Q.L = L;
    Q.s = m;
    Q.gates = (int64_t)taken.size();
    const uint64_t all = n >= 64 ? ~0ull : ((1ull << n) - 1);
    SuperPass sp;
    sp.mask = tile_mask;
    sp.pass_begin = 0;
    emit_pass(Q, recs, std::vector<int>(taken.begin(), taken.end()), tile_mask, all);
    sp.pass_end = 1;
    Q.supers.push_back(sp);
    Q.pass_gates.push_back(taken);
    Q.pass_op_begin.push_back((int64_t)Q.ops.size());
    return Q;
}

namespace {
void pauli2(int kind, cd *p) {
    const cd z(0, 0), one(1, 0), I(0, 1);
    if (kind == 1) { p[0] = z; p[1] = one; p[2] = one; p[3] = z; }
    else if (kind == 2) { p[0] = z; p[1] = -I; p[2] = I; p[3] = z; }
    else { p[0] = one; p[1] = z; p[2] = z; p[3] = -one; }
}
}  // namespace

bool pauli_commutes(const GateRec &g, int q, int kind) {
    if (!(((g.nmask | g.dmask) >> q) & 1)) return true;
    if (!can_conjugate_pauli(g, q, kind)) return false;
    GateRec h = g;
    conjugate_pauli(h, q, kind);
    if (h.nt != g.nt || h.cmask != g.cmask || h.t[0] != g.t[0] || (g.nt == 2 && h.t[1] != g.t[1])) return false;
    const int d = 1 << g.nt;
    for (int k = 0; k < d * d; ++k)
        if (h.u[k] != g.u[k]) return false;  // Pauli entries are 0, +-1, +-i: exact
    return true;
}

bool can_conjugate_pauli(const GateRec &g, int q, int kind) {
    if (!((g.cmask >> q) & 1) || kind == 3) return true;  // targets always; Z commutes with a control
    return g.diag && g.nt == 1 && popc(g.cmask) == 1;    // C-diag(d0,d1) -> diag over (q, t) with q flipped
}

void conjugate_pauli(GateRec &g, int q, int kind) {
    if ((g.cmask >> q) & 1) {
        if (kind == 3) return;
        // X_q C_q-D X_q = D applied where q = 0: a 2-qubit diagonal over (q, t)
        const cd d0 = g.u[0], d1 = g.u[3];
        GateRec h;
        h.nt = 2;
        h.t[0] = q;
        h.t[1] = g.t[0];
        for (int k = 0; k < 16; ++k) h.u[k] = 0;
        h.u[0] = d0;
        h.u[5] = d1;
        h.u[10] = h.u[15] = 1;
        h.cmask = 0;
        h.diag = true;
        h.nmask = 0;
        h.dmask = (1ull << q) | (1ull << g.t[0]);
        g = h;
        return;
    }
    int pos = -1;
    for (int k = 0; k < g.nt; ++k)
        if (g.t[k] == q) pos = k;
    if (pos < 0) return;
    cd p[4];
    pauli2(kind, p);
    const int d = 1 << g.nt;
    // full Pauli on the gate's index space: bit (nt-1-pos) of the row/column index
    const int bit = g.nt - 1 - pos;
    auto P = [&](int r, int c) -> cd {
        if ((r & ~(1 << bit)) != (c & ~(1 << bit))) return cd(0, 0);
        return p[2 * ((r >> bit) & 1) + ((c >> bit) & 1)];
    };
    cd t[16], u2[16];
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            cd s(0, 0);
            for (int k = 0; k < d; ++k) s += g.u[r * d + k] * P(k, c);
            t[r * d + c] = s;
        }
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            cd s(0, 0);
            for (int k = 0; k < d; ++k) s += P(r, k) * t[k * d + c];
            u2[r * d + c] = s;
        }
    bool diag = true;
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            g.u[r * d + c] = u2[r * d + c];
            if (r != c && u2[r * d + c] != cd(0, 0)) diag = false;
        }
    uint64_t tmask = 0;
    for (int k = 0; k < g.nt; ++k) tmask |= 1ull << g.t[k];
    g.diag = diag;
    g.nmask = diag ? 0 : tmask;
    g.dmask = g.cmask | (diag ? tmask : 0);
}

Plan rebuild_with_pass_r(const Plan &B, const std::vector<int> &rs) {
    Plan P;
    P.recs = B.recs;
    P.n = B.n;
    P.m = B.m;
    P.L = B.L;
    P.s = B.s;
    P.pass_budget = B.pass_budget;
    P.gates = B.gates;
    P.relabelled = B.relabelled;
    P.r = 0;
    for (int r : rs) P.r = std::max(P.r, r);
    const std::vector<GateRec> recs = relabel_swaps(B.recs, B.n);
    const uint64_t all = B.n >= 64 ? ~0ull : ((1ull << B.n) - 1);
    for (size_t k = 0; k < B.passes.size(); ++k) {
        SuperPass spp;
        spp.mask = B.passes[k].tile_mask;
        spp.pass_begin = (int32_t)P.passes.size();
        emit_pass(P, recs, std::vector<int>(B.pass_gates[k].begin(), B.pass_gates[k].end()), B.passes[k].tile_mask,
                  all, rs[k]);
        P.pass_gates.push_back(B.pass_gates[k]);
        spp.pass_end = (int32_t)P.passes.size();
        P.supers.push_back(spp);
    }
    P.pass_op_begin.push_back((int64_t)P.ops.size());
    return P;
}

int split_product_prefix(const std::vector<GateRec> &recs, int n, std::vector<GateRec> &kept, std::vector<cd> &prefix) {
    prefix.assign(4 * (size_t)n, cd(0.0));
    for (int q = 0; q < n; ++q) prefix[4 * q] = prefix[4 * q + 3] = cd(1.0);
    uint64_t blocked = 0;
    int absorbed = 0;
    kept.clear();
    for (const GateRec &g : recs) {
        const uint64_t touch = g.cmask | (1ull << g.t[0]) | (g.nt == 2 ? 1ull << g.t[1] : 0ull);
        if (g.nt == 1 && g.cmask == 0 && !((blocked >> g.t[0]) & 1)) {
            // A_q <- U A_q (U acts after the gates already absorbed on q)
            cd *a = &prefix[4 * g.t[0]];
            const cd a0 = a[0], a1 = a[1], a2 = a[2], a3 = a[3];
            a[0] = g.u[0] * a0 + g.u[1] * a2;
            a[1] = g.u[0] * a1 + g.u[1] * a3;
            a[2] = g.u[2] * a0 + g.u[3] * a2;
            a[3] = g.u[2] * a1 + g.u[3] * a3;
            ++absorbed;
            continue;
        }
        blocked |= touch;
        kept.push_back(g);
    }
    return absorbed;
}

void product_tables(const Plan &P, uint64_t basis, const std::vector<int> &regs, std::vector<cd> &tab) {
    const int n = P.n, G = (n + 4) / 5;
    std::vector<cd> v(2 * (size_t)n);
    for (int q = 0; q < n; ++q) {
        const int b = (int)((basis >> q) & 1);
        v[2 * q] = P.prefix[4 * q + b];          // column b_q of A_q
        v[2 * q + 1] = P.prefix[4 * q + 2 + b];
    }
    uint64_t regmask = 0;
    for (int q : regs) regmask |= 1ull << q;
    tab.assign(32 * (size_t)G + 2 * regs.size(), cd(1.0));
    for (int g = 0; g < G; ++g)
        for (int x = 0; x < 32; ++x) {
            cd f(1.0);
            for (int j = 0; j < 5; ++j) {
                const int q = 5 * g + j;
                if (q >= n) break;
                const int bit = (x >> j) & 1;
                if ((regmask >> q) & 1) {
                    if (bit) f = cd(0.0);  // register bits are zero in the thread's base index
                } else {
                    f *= v[2 * q + bit];
                }
            }
            tab[32 * g + x] = f;
        }
    for (size_t k = 0; k < regs.size(); ++k) {
        tab[32 * G + 2 * k] = v[2 * regs[k]];
        tab[32 * G + 2 * k + 1] = v[2 * regs[k] + 1];
    }
}

// Two-level schedule.  A SUPER-PASS selects s "super-tile" qubits S (greedy
// absorption with capacity s); its gates are then split into ordinary passes
// whose tiles lie inside S.  The executor runs all inner passes of a
// super-pass on one L2-resident super-tile (2^s amplitudes with the other
// qubits fixed) before moving to the next, so HBM sees one read + one write
// per super-pass while the inner passes stream through L2.  s >= n keeps the
// whole state in one super-tile; s == m degenerates to one pass per
// super-pass.
Plan build_plan(const std::vector<GateRec> &recs_in, int n, int m, int r, int L, int s) {
    Plan P;
    P.recs = recs_in;
    if (const char *b = std::getenv("QSV_PASS_BUDGET")) P.pass_budget = std::atof(b);
    P.n = n;
    P.m = m;
    P.r = r;
    P.L = L;
    P.s = std::max(m, std::min(s, n));
    P.gates = (int64_t)recs_in.size();
    const std::vector<GateRec> recs = relabel_swaps(recs_in, n);
    P.relabelled = recs.size() != recs_in.size();
    const uint64_t low = L > 0 ? ((1ull << L) - 1) : 0;
    const uint64_t all = n >= 64 ? ~0ull : ((1ull << n) - 1);

    std::vector<int> remaining(recs.size());
    for (size_t i = 0; i < recs.size(); ++i) remaining[i] = (int)i;

    if (P.s == m) {
        // flat schedule (no L2 super-tiles): one pass per super-pass entry
        std::vector<std::vector<int>> pass_gates;
        std::vector<uint64_t> pass_res;
        const bool search = !std::getenv("QSV_TILE_SEARCH") || std::atoi(std::getenv("QSV_TILE_SEARCH")) != 0;
        while (!remaining.empty()) {
            Absorber tile;
            tile.resident = low;
            tile.capacity = m;
            tile.budget = P.pass_budget;
            std::vector<int> taken, deferred;
            for (int gi : remaining) (tile.offer(recs[gi]) ? taken : deferred).push_back(gi);
            uint64_t res = tile.resident;
            if (search && P.pass_budget <= 0) {
                res = search_tile(recs, remaining, padded_tile(res, all, n, m), low, n);
                // look-ahead over 32 candidate tiles (n=32 RQC: 10 -> 8 passes; C2,
                // QFT, C5 unchanged; 32 and 100 candidates give identical plans on 14
                // C2/C3/C4/C5 circuits at half the planning time); QSV_PLAN_ROLLOUT=0
                // keeps the greedy tiles
                const int rollout = std::getenv("QSV_PLAN_ROLLOUT") ? std::atoi(std::getenv("QSV_PLAN_ROLLOUT")) : 32;
                if (rollout > 0) res = lookahead_tile(recs, remaining, res, low, all, n, m, rollout);
                taken.clear();
                deferred.clear();
                scan_fixed_tile(recs, remaining, res, &taken, &deferred);
            }
            pass_gates.push_back(taken);
            pass_res.push_back(res);
            remaining.swap(deferred);
        }
        balance_passes(recs, pass_gates, pass_res, all, n, m);
        for (size_t k = 0; k < pass_gates.size(); ++k) {
            if (pass_gates[k].empty()) continue;
            SuperPass spp;
            spp.mask = padded_tile(pass_res[k], all, n, m);
            spp.pass_begin = (int32_t)P.passes.size();
            emit_pass(P, recs, pass_gates[k], pass_res[k], all);
            P.pass_gates.emplace_back(pass_gates[k].begin(), pass_gates[k].end());
            spp.pass_end = (int32_t)P.passes.size();
            P.supers.push_back(spp);
        }
    }

    while (!remaining.empty()) {
        Absorber sup;
        sup.resident = low;
        sup.capacity = P.s;
        std::vector<int> s_taken, s_def;
        for (int gi : remaining) (sup.offer(recs[gi]) ? s_taken : s_def).push_back(gi);
        uint64_t smask = sup.resident;
        for (int q = 0; q < n && popc(smask) < P.s; ++q) smask |= 1ull << q;
        smask &= all;

        SuperPass spp;
        spp.mask = smask;
        spp.pass_begin = (int32_t)P.passes.size();
        std::vector<int> rem = s_taken;
        std::vector<std::vector<int>> pass_gates;
        std::vector<uint64_t> pass_res;
        while (!rem.empty()) {
            Absorber tile;
            tile.resident = low;
            tile.capacity = m;
            tile.budget = P.pass_budget;
            std::vector<int> taken, deferred;
            for (int gi : rem) (tile.offer(recs[gi]) ? taken : deferred).push_back(gi);
            pass_gates.push_back(taken);
            pass_res.push_back(tile.resident);
            rem.swap(deferred);
        }
        balance_passes(recs, pass_gates, pass_res, smask, n, m);
        for (size_t k = 0; k < pass_gates.size(); ++k)
            if (!pass_gates[k].empty()) {
                emit_pass(P, recs, pass_gates[k], pass_res[k], smask);
                P.pass_gates.emplace_back(pass_gates[k].begin(), pass_gates[k].end());
            }
        spp.pass_end = (int32_t)P.passes.size();
        P.supers.push_back(spp);
        remaining.swap(s_def);
    }
    P.pass_op_begin.push_back((int64_t)P.ops.size());
    return P;
}

PlanObjectiveScope::PlanObjectiveScope(int objective) : saved(t_plan_objective) { t_plan_objective = objective; }
PlanObjectiveScope::~PlanObjectiveScope() { t_plan_objective = saved; }

}  // namespace qsv
