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
#include <bit>
#include <cstring>

namespace qsv {

static inline int popc(uint64_t x) { return std::popcount(x); }

void resolve_options(const qsv_options *opt, int n, int &m, int &r, int &L) {
    m = (opt && opt->tile_qubits > 0) ? opt->tile_qubits : 12;
    r = (opt && opt->reg_qubits > 0) ? opt->reg_qubits : 4;
    L = (opt && opt->low_qubits > 0) ? opt->low_qubits : 5;
    m = std::min(std::min(m, kMaxTileQubits), n);
    r = std::max(std::min(std::min(r, kMaxRegQubits), m), std::min(2, m));
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

struct Absorber {
    uint64_t resident = 0;  // qubits currently resident (tile or registers)
    int capacity = 0;
    uint64_t blockN = 0, blockD = 0;

    // true when gate g is taken
    bool offer(const GateRec &g) {
        const uint64_t touched = g.nmask | g.dmask;
        bool blocked = (touched & blockN) || (g.nmask & blockD);
        if (!blocked) {
            const uint64_t need = g.nmask & ~resident;
            if (popc(resident | need) <= capacity) {
                resident |= need;
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

// Op as seen in global-qubit terms while a stage is being assembled.
struct StageOp {
    int kind;
    int qa, qb;
    uint64_t cmask;
    cd m[16];
};

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

// Appends `o` to the stage, fusing it into an earlier single-qubit op on the
// same target with the same controls when every op in between commutes with it.
void append_fused(std::vector<StageOp> &ops, const StageOp &o) {
    if (o.kind == QSV_OP_MAT1 || o.kind == QSV_OP_DIAG1) {
        const uint64_t q = 1ull << o.qa;
        const bool o_diag = o.kind == QSV_OP_DIAG1;
        for (int k = (int)ops.size() - 1; k >= 0; --k) {
            StageOp &p = ops[k];
            const bool same = (p.kind == QSV_OP_MAT1 || p.kind == QSV_OP_DIAG1) && p.qa == o.qa &&
                              p.cmask == o.cmask;
            if (same) {
                cd a[4], b[4], r[4];
                auto full = [](const StageOp &x, cd *dst) {
                    if (x.kind == QSV_OP_DIAG1) {
                        dst[0] = x.m[0]; dst[1] = 0; dst[2] = 0; dst[3] = x.m[1];
                    } else {
                        for (int i = 0; i < 4; ++i) dst[i] = x.m[i];
                    }
                };
                full(p, a);
                full(o, b);
                mul2(b, a, r);
                if (p.kind == QSV_OP_DIAG1 && o_diag) {
                    p.m[0] = r[0];
                    p.m[1] = r[3];
                } else {
                    p.kind = QSV_OP_MAT1;
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

}  // namespace

Plan build_plan(const std::vector<GateRec> &recs, int n, int m, int r, int L) {
    Plan P;
    P.n = n;
    P.m = m;
    P.r = r;
    P.L = L;
    P.gates = (int64_t)recs.size();
    const uint64_t low = L > 0 ? ((1ull << L) - 1) : 0;

    std::vector<int> remaining(recs.size());
    for (size_t i = 0; i < recs.size(); ++i) remaining[i] = (int)i;

    while (!remaining.empty()) {
        Absorber tile;
        tile.resident = low;
        tile.capacity = m;
        std::vector<int> taken, deferred;
        for (int gi : remaining) (tile.offer(recs[gi]) ? taken : deferred).push_back(gi);

        // pad the tile with the lowest unused qubits (coalescing)
        uint64_t tmask = tile.resident;
        for (int q = 0; q < n && popc(tmask) < m; ++q) tmask |= 1ull << q;

        DevPass dp;
        std::memset(&dp, 0, sizeof(dp));
        dp.tile_mask = tmask;
        dp.m = m;
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

            std::vector<StageOp> sops;
            for (int gi : st_taken) append_fused(sops, make_op(recs[gi]));

            DevStage ds;
            std::memset(&ds, 0, sizeof(ds));
            int k = 0;
            int32_t regpos_of_local[64];
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
                DevOp d;
                std::memset(&d, 0, sizeof(d));
                d.kind = o.kind;
                d.qa = o.qa;
                d.qb = o.qb;
                uint64_t cl = 0, ce = 0;
                for (int q = 0; q < n; ++q) {
                    if (!((o.cmask >> q) & 1)) continue;
                    const int lb = local_bit(tmask, q);
                    if (lb >= 0) cl |= 1ull << lb;
                    else ce |= 1ull << q;
                }
                d.cmask_local = (uint32_t)cl;
                d.cmask_ext = ce;
                if (o.kind == QSV_OP_MAT1 || o.kind == QSV_OP_MAT2) {
                    d.a = regpos_of_local[local_bit(tmask, o.qa)];
                    d.b = o.kind == QSV_OP_MAT2 ? regpos_of_local[local_bit(tmask, o.qb)] : -1;
                } else {
                    d.a = local_bit(tmask, o.qa);
                    d.b = o.kind == QSV_OP_DIAG2 ? local_bit(tmask, o.qb) : -1;
                }
                const int cnt = o.kind == QSV_OP_MAT2 ? 16 : (o.kind == QSV_OP_DIAG1 ? 2 : 4);
                for (int i = 0; i < cnt; ++i) {
                    d.m[2 * i] = o.m[i].real();
                    d.m[2 * i + 1] = o.m[i].imag();
                }
                P.ops.push_back(d);
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
        remaining.swap(deferred);
    }
    P.pass_op_begin.push_back((int64_t)P.ops.size());
    return P;
}

}  // namespace qsv
