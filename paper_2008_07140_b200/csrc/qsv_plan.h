// Host-side gate scheduler/fuser of libqsv (no reference counterpart: the
// reference applies one full-state sweep per gate, statevector.py:425-426, and
// SPEC.md:115 rules fusion out).  Shared by the CUDA launcher (qsv_api.cu).
//
// Execution model the plan targets:
//   * a PASS streams the whole state through shared memory once: every CTA
//     owns a tile of 2^m amplitudes whose index bits over the pass's m "tile
//     qubits" vary and whose other bits are fixed (the tile base);
//   * inside a pass, STAGES hold 2^r amplitudes per thread in registers over r
//     "register qubits"; between stages the tile is re-laid out through shared
//     memory;
//   * an op is applied to register-resident amplitudes: non-diagonal targets
//     must be register qubits, while diagonal factors and controls may sit on
//     any qubit (tile-local bits come from the amplitude's local index, the
//     other bits from the tile base) - so CZ/T/CR/RZ never cost residency.
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qsv.h"

namespace qsv {

using cd = std::complex<double>;

constexpr int kMaxTileQubits = 13;  // 2^13 * 16 B = 128 KiB shared memory
constexpr int kMaxRegQubits = 4;    // 16 amplitudes (64 registers) per thread
constexpr int kLoTabBits = 6;       // local-index -> offset tables: 6 low bits ...
constexpr int kHiTabBits = kMaxTileQubits - kLoTabBits;  // ... + 7 high bits

// Device-side op record (16-byte aligned; read uniformly by every thread).
struct DevOp {
    int32_t kind;   // QSV_OP_*
    int32_t a, b;   // MAT: register positions (a = MSB target); DIAG: local bits or -1
    int32_t qa, qb; // DIAG: global qubits (used when the local bit is -1)
    uint32_t cmask_local;  // controls on tile-local bits
    uint64_t cmask_ext;    // controls on qubits outside the tile (per-CTA test)
    double m[32];          // row-major complex matrix / diagonal entries
};

struct DevStage {
    uint32_t reg_local_mask;  // local bits held in registers
    int32_t op_begin, op_end;
    int32_t rb[kMaxRegQubits];  // register position k <-> local bit rb[k]
    int32_t pad;
};

struct DevPass {
    uint64_t tile_mask;
    int32_t m, stage_begin, stage_end, pad;
    int32_t tq[kMaxTileQubits + 3];         // local bit j <-> global qubit tq[j]
    uint64_t lo_tab[1 << kLoTabBits];       // offset of local bits [0,6)
    uint64_t hi_tab[1 << kHiTabBits];       // offset of local bits [6,m)
};

struct GateRec {
    int nt = 1;
    int t[2] = {0, 0};
    uint64_t cmask = 0;
    cd u[16];
    bool diag = false;
    uint64_t nmask = 0;  // qubits acted on non-diagonally (targets of a non-diagonal gate)
    uint64_t dmask = 0;  // qubits acted on diagonally (controls, targets of diagonal gates)
};

struct Plan {
    int n = 0, m = 0, r = 0, L = 0;
    int64_t gates = 0;
    std::vector<DevPass> passes;
    std::vector<DevStage> stages;
    std::vector<DevOp> ops;
    std::vector<int32_t> op_stage;        // stage index (within pass) of every op
    std::vector<uint64_t> stage_regs;     // global register-qubit mask per stage
    std::vector<int64_t> pass_op_begin;   // first op of every pass (+ sentinel)
    // device copies (owned by the launcher, lazily uploaded)
    void *d_passes = nullptr, *d_stages = nullptr, *d_ops = nullptr;
    int device = -1;
};

// Validates and classifies gate records; returns QSV_OK or an error status (msg set).
int to_records(const qsv_gate *gates, int64_t n_gates, int n_qubits, std::vector<GateRec> &out,
               std::string &msg);

// Builds the fused schedule.  m, r, L already clamped to the state size.
Plan build_plan(const std::vector<GateRec> &recs, int n, int m, int r, int L);

void resolve_options(const qsv_options *opt, int n, int &m, int &r, int &L);

}  // namespace qsv
