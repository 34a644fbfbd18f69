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
constexpr int kMaxRegQubits = 5;    // up to 32 amplitudes per thread (R = 5: specialised kernels only)
constexpr int kLoTabBits = 6;       // local-index -> offset tables: 6 low bits ...
constexpr int kHiTabBits = kMaxTileQubits - kLoTabBits;  // ... + 7 high bits

// Device op kinds (internal; the exported qsv_op_info uses QSV_OP_* in global terms).
enum : int32_t { K_MAT1 = 1, K_MAT2 = 2, K_DIAG = 3 };
// MAT1 variants: structure of the 2x2 decides the FP64 work per amplitude
enum : int32_t { V_GEN = 0, V_REAL = 1, V_RXL = 2 };  // RXL: real diagonal, imaginary off-diagonal
enum : int32_t { V_PERM = 1 };                        // MAT2: one nonzero per row (SWAP, iSWAP, CNOT, ...)
// DIAG variants: which of the (<=2) diagonal qubits are register-resident
enum : int32_t { D_NONE = 0, D_A = 1, D_B = 2, D_AB = 3 };
constexpr int32_t kScalarExt = 64;   // scalar descriptor >= 64: external global qubit (desc - 64)

// Device-side op record (16-byte aligned; read uniformly by every thread).  Each
// qubit an op touches is classified at plan time as a register position (varies
// across a thread's 2^R amplitudes), a thread bit (a tile-local bit fixed per
// thread in this stage) or an external bit (fixed per tile), so the kernel
// never tests index bits per amplitude for anything but register positions.
struct alignas(16) DevOp {
    // code: kind | var << 4 | a << 8 | b << 12 | modes << 16 | src << 24
    //   a, b   register positions (MAT targets, a = MSB; DIAG register qubits), 15 = none
    //   modes  DIAG: 2 bits per entry d[e]: 0 exactly 1 (skip), 1 exactly -1 (sign flip), 2 general
    //   src    MAT2/PERM: 2 bits per output row r = input column feeding it
    uint32_t code;
    uint32_t rs;    // rc (controls on register positions, 8 bits) | sa << 8 | sb << 16 (DIAG scalar qubits)
    uint32_t tc;    // controls on thread bits (tile-local bit mask)
    uint32_t pad0;
    uint64_t ec;    // controls on external qubits (global mask)
    uint64_t pad1;
    double m[32];   // MAT1: 2x2; MAT2: 4x4 (PERM: m[2r] = phase of row r); DIAG: d[4] over (bitA, bitB)
};
constexpr uint32_t kNoReg = 15;
constexpr uint32_t kNoScalar = 0xff;  // scalar descriptor: none; [0,32) tile-local bit; [64,128) external qubit - 64

// Op in global-qubit terms (kept host-side for export/validation).
struct GlobalOp {
    int kind;  // QSV_OP_*
    int qa, qb;
    uint64_t cmask;
    std::complex<double> m[16];
};

struct DevStage {
    uint32_t reg_local_mask;  // local bits held in registers
    int32_t op_begin, op_end;
    int32_t rb[kMaxRegQubits];  // register position k <-> local bit rb[k]
    int32_t pad;
};

struct alignas(16) DevPass {
    uint64_t tile_mask;
    int32_t m, stage_begin, stage_end, r;  // r: register qubits of this pass's stages
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

// A super-pass: inner passes [pass_begin, pass_end) whose tiles lie inside
// the super-tile qubits `mask` (executed super-tile by super-tile through L2).
struct SuperPass {
    uint64_t mask = 0;
    int32_t pass_begin = 0, pass_end = 0;
};

struct Plan {
    int n = 0, m = 0, r = 0, L = 0, s = 0;
    std::vector<GateRec> recs;  // the gate records the plan was built from
    double pass_budget = 0;     // cap on estimated FP64 work per pass (0: none)
    std::vector<SuperPass> supers;
    int64_t gates = 0;
    std::vector<DevPass> passes;
    std::vector<DevStage> stages;
    std::vector<DevOp> ops;
    std::vector<int32_t> op_stage;        // stage index (within pass) of every op
    std::vector<GlobalOp> gops;           // every op in global-qubit terms
    std::vector<uint64_t> stage_regs;     // global register-qubit mask per stage
    std::vector<int64_t> pass_op_begin;   // first op of every pass (+ sentinel)
    std::vector<std::vector<int32_t>> pass_gates;  // gate records (indices into recs) of every pass, in order
    bool relabelled = false;              // SWAPs were folded into a qubit relabelling (indices shifted)
    // device copies (owned by the launcher, lazily uploaded)
    void *d_passes = nullptr, *d_stages = nullptr, *d_ops = nullptr;
    int device = -1;
    // specialised kernels (qsv_jit.cpp), one CUfunction per pass
    std::vector<void *> jit_funcs;
    std::vector<int> jit_grids;
    std::vector<int> jit_gangs;  // tiles per CTA of each pass kernel
    std::vector<void *> jit_super_funcs;  // per super-pass (nullptr: run its inner passes flat)
    std::vector<int> jit_super_grids;
    std::vector<int> super_use;  // cost-model choice per super-pass (jit_choose_supers)
    // deferred uniform scale carried into each pass by the specialised kernels
    // (+ the plan's output, always 1); filled on first use by qsv_jit.cpp
    mutable std::vector<double> jit_scale_in;
    int jit_device = -1;
    // kernels of a plan still compiling asynchronously (jit_start_async): per-pass
    // sources and the passes loaded so far
    std::vector<std::string> jit_part_src;
    std::vector<void *> jit_part_funcs;
    std::vector<int> jit_part_grids;
    // product-state start (qsv_options.product_start): the leading single-qubit
    // gates of every qubit (each before any other gate touching that qubit) are
    // not in `recs`; they map a basis state |b> to the product state
    // (x)_q prefix_q e_{b_q}, which pass 0 synthesises from host-built factor
    // tables instead of reading the state.  Such a plan only runs on a state
    // holding a pending basis index (qsv_set_basis).
    bool product = false;
    std::vector<cd> prefix;  // 4 per qubit: row-major 2x2 product of the absorbed gates
};

// Splits `recs` into the leading uncontrolled single-qubit gates of each qubit
// (multiplied into prefix[4q..4q+3]) and the rest (`kept`, program order).
// Returns the number of absorbed gates.
int split_product_prefix(const std::vector<GateRec> &recs, int n, std::vector<GateRec> &kept, std::vector<cd> &prefix);

// Factor tables of a product-start plan for basis index `basis`: for every
// group g of 5 index bits, tab[32 g + x] = prod over the group's qubits q that are
// not in `regs` of v_q[bit of x], then for every register qubit regs[k] the pair
// tab[32 G + 2k + b] = v_{regs[k]}[b]  (v_q = prefix_q e_{b_q}, G = ceil(n / 5)).
void product_tables(const Plan &P, uint64_t basis, const std::vector<int> &regs, std::vector<cd> &tab);

// Validates and classifies gate records; returns QSV_OK or an error status (msg set).
int to_records(const qsv_gate *gates, int64_t n_gates, int n_qubits, std::vector<GateRec> &out,
               std::string &msg);

// Builds the fused schedule.  m, r, L already clamped to the state size.
Plan build_plan(const std::vector<GateRec> &recs, int n, int m, int r, int L, int s);
// Look-ahead objective of the plans built on this thread while the scope lives
// (qsv_options.plan_objective: 1 = fewest passes, otherwise modeled time).
struct PlanObjectiveScope {
    explicit PlanObjectiveScope(int objective);
    ~PlanObjectiveScope();
    int saved;
};

// The same passes (tiles and gate sets) as the flat plan B, each re-staged with
// its own number of register qubits rs[k] (P.r = max).
Plan rebuild_with_pass_r(const Plan &B, const std::vector<int> &rs);

// register qubits of pass pi's stages
inline int pass_r(const Plan &P, int pi) {
    const int r = P.passes[pi].r;
    return r > 0 ? r : P.r;
}

// One pass over `tile_mask` applying recs[taken] (program order) with r
// register qubits: the interpreted kernel's tables for a pass whose gates
// differ from a compiled plan's (noisy trajectories, qsv_plan_execute_paulis).
Plan build_single_pass(const std::vector<GateRec> &recs, const std::vector<int32_t> &taken, uint64_t tile_mask, int n,
                       int m, int r, int L);

// P U P for a Pauli (1 X, 2 Y, 3 Z) on qubit q: gate g as seen when the Pauli is
// moved across it.  False when the result is no gate record (a non-diagonal
// gate, or a multi-controlled one, controlled by q, conjugated by X or Y).
bool can_conjugate_pauli(const GateRec &g, int q, int kind);
void conjugate_pauli(GateRec &g, int q, int kind);
// P G P == G exactly (the Pauli moves across G without changing it)
bool pauli_commutes(const GateRec &g, int q, int kind);

// SWAP gates folded into a logical->physical qubit map (see qsv_plan.cpp).
std::vector<GateRec> relabel_swaps(const std::vector<GateRec> &recs, int n);

void resolve_options(const qsv_options *opt, int n, int &m, int &r, int &L, int &s);

// Distributed layout: segments of the stream that each run with one fixed set of
// `capacity` local qubits (see qsv_plan.cpp).  gate_seg[i] = segment of gate i.
int plan_segments(const std::vector<GateRec> &recs, int n, int capacity, uint64_t init_local, bool free_initial,
                  std::vector<int32_t> &gate_seg, std::vector<uint64_t> &seg_local);

}  // namespace qsv
