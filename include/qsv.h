/*
 * qsv.h - C ABI of libqsv.so, the B200-native full-amplitude state-vector engine.
 *
 * The reference (qcsim 0.1.0, pure Python + numba) has no plugin registry; its
 * seam is function level.  Each entry point below replaces one
 * reference function; the Python host package paper_2008_07140_b200 binds them
 * with ctypes (see INTEGRATION.md for the binding a maintainer would add).
 *
 *   qsv_create / qsv_set_basis  <- statevector.init_state          statevector.py:52-65
 *                                  (+ run_full initial_index)      statevector.py:421-423
 *   qsv_upload / qsv_download   <- StateVector(n, amps, ...)       statevector.py:32-36
 *                                  / StateVector.amplitudes reads
 *   qsv_apply_gate              <- _apply_gate (apply_single_qubit,
 *                                  apply_controlled, apply_two_qubit,
 *                                  apply_projector)                statevector.py:217-289
 *   qsv_run / qsv_plan_*        <- the run_full gate loop          statevector.py:425-426
 *                                  (fused + scheduled; no reference
 *                                  counterpart: SPEC.md:115 has no fusion)
 *   qsv_norm_sq                 <- StateVector.norm_sq             statevector.py:42-43
 *   qsv_prob_bit0               <- probability_bit0                statevector.py:292-295
 *   qsv_collapse                <- the collapse half of measure    statevector.py:305-307
 *   qsv_pmeasure                <- pmeasure                        statevector.py:311-328
 *   qsv_scale                   <- noise renormalisation           noise.py:219-221
 *   qsv_reduced_density         <- branch_probabilities            noise.py:145-185
 *
 * Conventions: amplitudes are complex128 (interleaved
 * re, im float64), index bit k <-> qubit k (little-endian).  Gate matrices are
 * row-major with the FIRST target as the matrix MSB (gates.py:3-4); controls
 * are a bit mask and act on the all-ones block only (gates.py:162-168).
 *
 * Every call returns 0 on success or a negative status whose class mirrors
 * qcsim/errors.py (see QSV_E_*); qsv_state_last_error(st) gives the message of the
 * last failed call on that handle (qsv_last_error() the calling thread's last one,
 * for calls without a handle).  Calls are
 * asynchronous on the state's stream except readouts, which synchronise.
 * There is no CPU execution path: without a CUDA device, state calls fail
 * with QSV_E_DEVICE.  The planning calls (qsv_plan_*) are pure host code.
 */
#ifndef QSV_H
#define QSV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSV_OK 0
#define QSV_E_PARSE (-2)           /* ParseError             (exit code 2) */
#define QSV_E_TOO_MANY_QUBITS (-3) /* TooManyQubits          (exit code 3) */
#define QSV_E_NUMERIC (-4)         /* NumericError           (exit code 4) */
#define QSV_E_DEVICE (-5)          /* CUDA / NCCL failure, no reference analogue */
#define QSV_E_UNSUPPORTED (-6)     /* UnsupportedGate        (exit code 2) */
#define QSV_E_DEGENERATE (-7)      /* DegenerateState        (exit code 4) */

#define QSV_MAX_QUBITS 63

typedef struct qsv_state qsv_state;
typedef struct qsv_plan qsv_plan;

/* One gate in controlled form: the record of gates.controlled_form (gates.py:150-159). */
typedef struct qsv_gate {
    int32_t n_targets;     /* 1 or 2 */
    int32_t targets[2];    /* targets[0] is the matrix MSB */
    uint64_t control_mask; /* bit q set <=> control on qubit q; must not overlap targets */
    double u[32];          /* row-major complex (re,im): 2x2 uses u[0..7], 4x4 u[0..31] */
} qsv_gate;

/* Scheduling knobs.  Zero means "library default". */
typedef struct qsv_options {
    int32_t fuse;        /* 0: one kernel per gate (reference-shaped, unfused)  1: fused passes */
    int32_t tile_qubits; /* m: qubits resident in one CTA tile (2^m amplitudes in shared memory) */
    int32_t reg_qubits;  /* r: qubits held in registers per stage (2^r amplitudes per thread) */
    int32_t low_qubits;  /* L: lowest qubits always in the tile (coalescing) */
    int32_t profile;     /* 1: time every launch with CUDA events (qsv_run_stats) */
    int32_t n_global;    /* sharded layout: top n_global qubits are global (not resident) */
    int32_t jit;         /* pass kernels: 0 auto (specialise when n >= 16), 1 always, -1 never
                            (specialised = runtime-generated CUDA compiled with NVRTC for sm_100a) */
    int32_t super_qubits; /* s: qubits of an L2-resident super-tile (2^s amplitudes; default 21) */
    int32_t product_start; /* 1: absorb every qubit's leading single-qubit gates into a product-state
                              start that the first pass synthesises (the plan then runs only on a
                              state holding a pending basis index, qsv_set_basis); -1: never;
                              0: auto - qsv_run uses it for a pending basis state with specialised
                              kernels, qsv_plan_create does not */
    int32_t plan_objective; /* what the scheduler's look-ahead minimises: 0 / 2 the summed modeled
                              pass time (balanced FP64 work per pass; default), 1 the number of
                              passes (front-loaded passes: faster for plans that carry Pauli errors,
                              qsv_plan_execute_paulis) */
} qsv_options;

typedef struct qsv_run_stats {
    int64_t gates;         /* gate records consumed */
    int64_t passes;        /* HBM passes executed (super-passes, or unfused gate kernels) */
    int64_t stages;        /* register stages (shared-memory round trips) inside passes */
    int64_t inner_passes;  /* tile passes (L2-resident inside a super-pass) */
    int64_t launches;      /* kernels launched by this call */
    double kernel_ms;      /* sum of event-timed launch durations (profile=1 only) */
    double max_launch_ms;  /* longest single launch (profile=1 only) */
    double algorithmic_bytes; /* per pass 2 * 16 * 2^n_local (16 * 2^n_local when it synthesises a basis input) */
    double plan_ms;        /* host time building schedules for this call (0 when the plan was cached) */
    double jit_ms;         /* host time specialising + compiling (NVRTC) / loading pass kernels */
    int64_t compiled_passes; /* passes of a cold call (kernels still compiling in the background) that
                                ran compiled; the others ran on the interpreted pass kernel */
} qsv_run_stats;

typedef struct qsv_plan_info {
    int32_t n_qubits, tile_qubits, reg_qubits, low_qubits;
    int64_t gates, passes, stages, ops;
    int32_t super_qubits;
    int32_t product_start; /* 1: the plan starts from a product state (qsv_options.product_start) */
    int64_t super_passes; /* HBM passes: each streams the state once through L2 */
} qsv_plan_info;

/* One fused pass: a tile of 2^m amplitudes over the qubits in tile_mask. */
typedef struct qsv_pass_info {
    uint64_t tile_mask;
    int32_t m;
    int32_t n_stages;
    int64_t n_ops;
    uint64_t super_mask;   /* qubits of the super-tile this pass runs inside */
    int64_t super_index;   /* which super-pass it belongs to */
} qsv_pass_info;

#define QSV_OP_MAT1 1  /* 2x2 on register position a               */
#define QSV_OP_MAT2 2  /* 4x4 on register positions a (MSB), b     */
#define QSV_OP_DIAG1 3 /* diag(d0,d1) on qubit qa                  */
#define QSV_OP_DIAG2 4 /* diag(d00,d01,d10,d11) on qubits qa (MSB), qb */

/* One operation of a pass, exported for inspection/validation (tests emulate it). */
typedef struct qsv_op_info {
    int32_t stage;         /* stage index inside the pass */
    int32_t kind;          /* QSV_OP_* */
    int32_t qa, qb;        /* global qubits acted on (qb = -1 when unused) */
    uint64_t control_mask; /* global control qubits */
    uint64_t stage_regs;   /* global qubits held in registers during this stage */
    double m[32];          /* MAT1: 2x2, MAT2: 4x4, DIAG1: d0,d1, DIAG2: d00..d11 (complex) */
} qsv_op_info;

const char *qsv_version(void);
const char *qsv_last_error(void);
/* message of the last failed call made on `st` (per handle: calls on other handles or
 * threads in between do not overwrite it); "" when none failed */
const char *qsv_state_last_error(const qsv_state *st);
/* The first qsv_run of a new circuit does not wait for NVRTC: its pass kernels compile on
 * background host threads while the passes run (compiled once ready, interpreted before;
 * qsv_run_stats.compiled_passes).  qsv_jit_wait blocks until no such compile is pending,
 * so the next call runs fully compiled. */
int qsv_jit_wait(void);
/* per-launch event times (ms) and algorithmic bytes of the last call on `st` that ran
 * with qsv_options.profile = 1 (bytes: 2 x 16 x 2^n per pass, 16 x 2^n for a pass that
 * synthesises its basis-state input); copies min(count, cap) entries */
int qsv_last_launches(const qsv_state *st, double *ms, double *bytes, int64_t cap, int64_t *count);
int qsv_device_count(int *out);

/* ---- state lifetime and data movement ---- */
int qsv_create(int n_qubits, int device, void *stream, qsv_state **out);
/* wraps caller-owned device memory (e.g. a torch tensor); its contents are left untouched */
int qsv_create_on(int n_qubits, int device, void *stream, void *device_amplitudes, qsv_state **out);
int qsv_destroy(qsv_state *st);
int qsv_device_ptr(qsv_state *st, void **out);
int qsv_set_basis(qsv_state *st, uint64_t index);
int qsv_upload(qsv_state *st, const void *host_c128, uint64_t offset, uint64_t count);
int qsv_download(qsv_state *st, void *host_c128, uint64_t offset, uint64_t count);
/* amplitude k of host_c128 -> index offset + k * stride, k < count (one 2-D copy): the start
 * amplitudes of batched trajectory blocks (noisy_batch.py) */
int qsv_upload_strided(qsv_state *st, const void *host_c128, uint64_t offset, uint64_t count, uint64_t stride);
/* enqueues the download on the state's stream and returns: `host_c128` must be
 * pinned and is complete after qsv_synchronize(st) (overlaps another state's
 * simulation; used by the batched run, statevector.run_batch) */
int qsv_download_async(qsv_state *st, void *host_c128, uint64_t offset, uint64_t count);
int qsv_synchronize(qsv_state *st);

/* ---- gate application ---- */
int qsv_apply_gate(qsv_state *st, const qsv_gate *gate);
int qsv_run(qsv_state *st, const qsv_gate *gates, int64_t n_gates, const qsv_options *opt,
            qsv_run_stats *stats);

/* ---- planning (host only; usable without a GPU) ---- */
int qsv_plan_create(const qsv_gate *gates, int64_t n_gates, int n_qubits, const qsv_options *opt,
                    qsv_plan **out);
int qsv_plan_destroy(qsv_plan *plan);
int qsv_plan_summary(const qsv_plan *plan, qsv_plan_info *out);
int qsv_plan_pass(const qsv_plan *plan, int64_t pass, qsv_pass_info *out);
int qsv_plan_op(const qsv_plan *plan, int64_t pass, int64_t op, qsv_op_info *out);
int qsv_plan_execute(qsv_state *st, qsv_plan *plan, const qsv_options *opt, qsv_run_stats *stats);
/* factor tables a product-start plan's first pass reads for basis index `basis` (complex,
 * interleaved re/im; count = entries): host code, used to run the host rendering in tests */
int qsv_plan_product_tables(const qsv_plan *plan, uint64_t basis, double *out, int64_t cap, int64_t *count);

/* source of the specialised (runtime-generated) kernel of one pass; copies at most
 * buf_size bytes (NUL-terminated) and reports the full size in *needed; host=1 renders the
 * same pass as plain C++ (used by the CPU tests to check the generator) */
int qsv_plan_kernel_source(const qsv_plan *plan, int64_t pass, int host, char *buf, int64_t buf_size,
                           int64_t *needed);
/* source of the exchange-out variant of one pass (qsv_run_exchange); host=1 renders it as C++
 * with signature (double2 *psi, u64 n_tiles, XDst xd) */
int qsv_plan_exchange_source(const qsv_plan *plan, int64_t pass, int host, uint64_t positions, char *buf,
                             int64_t buf_size, int64_t *needed);
/* source of the persistent kernel of one super-pass (all its inner passes on L2-resident
 * super-tiles, grid barrier in between); host=1 renders it as plain C++ */
int qsv_plan_super_source(const qsv_plan *plan, int64_t super_pass, int host, char *buf, int64_t buf_size,
                          int64_t *needed);
/* FP64 instructions per amplitude the specialised kernel of one pass executes (cost model) */
int qsv_plan_pass_cost(const qsv_plan *plan, int64_t pass, double *fp64_per_amp);
/* distributed layout (sharded state, n_local of n_qubits qubits local per rank): cut the stream
 * into SEGMENTS that each run with one fixed set of n_local local logical qubits; between
 * segments the leaving/entering qubits are exchanged (global<->local qubit swap).
 * gate_segment[n_gates] receives the segment of every gate, segment_local[n_gates] the local
 * qubit mask of every segment, *n_segments their number.  initial_local = current local set;
 * free_initial=1 lets the first segment pick its own (basis-state input).  No reference
 * counterpart (the reference has no distributed mode). */
int qsv_plan_segments(const qsv_gate *gates, int64_t n_gates, int n_qubits, int n_local, uint64_t initial_local,
                      int free_initial, int32_t *gate_segment, uint64_t *segment_local, int64_t *n_segments);
/* compile CUDA source for sm_100a with NVRTC (no GPU needed); *cubin_bytes = image size */
int qsv_jit_compile(const char *src, int64_t *cubin_bytes);

/* ---- peer exchange for the sharded layout (one process per GPU, NVLink copy engines) ----
 * No reference counterpart (the reference is single-node).  The global<->local
 * qubit swap of distributed.py pushes contiguous blocks into the peers' receive buffers. */
/* CUDA IPC handle (64 bytes) of the allocation holding device_ptr, and device_ptr's byte offset in it */
int qsv_ipc_mem_handle(void *device_ptr, void *handle64, uint64_t *offset);
/* maps a peer allocation into this process on `device`; *out = base + offset */
int qsv_ipc_mem_open(const void *handle64, uint64_t offset, int device, void **out);
int qsv_ipc_mem_close(void *mapped);
/* Global<->local qubit swap FUSED into the last pass of a gate run: the run's fused passes execute
 * as in qsv_run, except that the last one stores every output amplitude straight into the
 * receive buffer of the rank selected by its bits at `positions` (dst[value], a peer allocation
 * mapped with qsv_ipc_mem_open, or this rank's own), at the same offset with those bits replaced
 * by `self_bits` (this rank's global bits deposited at `positions`).  The state buffer itself is
 * left stale.  QSV_E_UNSUPPORTED without specialised kernels or with super-passes (the caller then
 * runs qsv_run and copies). */
typedef struct qsv_exchange {
    uint64_t positions;
    uint64_t self_bits;
    uint64_t dst[8];
} qsv_exchange;
int qsv_run_exchange(qsv_state *st, const qsv_gate *gates, int64_t n_gates, const qsv_options *opt,
                     const qsv_exchange *ex, qsv_run_stats *stats);
/* *out = 1 when qsv_run_exchange can fuse an exchange at `positions` into this run (plans it; the
 * plan is cached for the following qsv_run_exchange).  Ranks agree collectively before fusing. */
int qsv_exchange_fusable(qsv_state *st, const qsv_gate *gates, int64_t n_gates, const qsv_options *opt,
                         uint64_t positions, int *out);
/* asynchronous copy between any two device pointers (UVA; peer pointers go over NVLink) */
int qsv_copy_async(void *dst, const void *src, uint64_t bytes, void *stream);

/* ---- noisy trajectories on a compiled plan ----
 * One Pauli error (1 = X, 2 = Y, 3 = Z) on `qubit` acting right BEFORE gate record `gate` of the
 * plan's gate list (gate == n_gates: after the last gate): the explicit X/Y/Z insertion of a
 * pre-sampled depolarising trajectory (noise.py:188-222 semantics, workloads.py).  The reference
 * re-runs every trajectory gate by gate (statevector.py:343-357). */
typedef struct qsv_pauli {
    int64_t gate;
    int32_t qubit;
    int32_t kind;
} qsv_pauli;
/* Runs `plan` with Pauli errors inserted, reusing the plan's compiled pass kernels: every error
 * is moved to a pass boundary (gates on its qubit that it crosses are replaced by their Pauli
 * conjugates; the boundary chosen crosses as few passes' gates as possible), applied there as a
 * Pauli-string kernel, and only passes holding conjugated gates run through the interpreted
 * kernel.  QSV_E_UNSUPPORTED when the plan relabelled SWAPs or uses super-passes. */
int qsv_plan_execute_paulis(qsv_state *st, qsv_plan *plan, const qsv_pauli *paulis, int64_t n_paulis,
                            const qsv_options *opt, qsv_run_stats *stats);
/* qsv_plan_execute_paulis (n_paulis may be 0) followed by the probe table (1..4 qubits, first listed =
 * MSB, statevector.py:311-328 semantics) of the final state, written to DEVICE memory on the state's
 * stream.  When the plan's last pass runs compiled with nothing after it, that pass accumulates the
 * table while it stores (no extra read of the state); otherwise pmeasure runs after it. */
int qsv_plan_execute_probe(qsv_state *st, qsv_plan *plan, const qsv_pauli *paulis, int64_t n_paulis,
                           const int32_t *probe_qubits_msb_first, int m, double *device_table, const qsv_options *opt,
                           qsv_run_stats *stats);
/* host only (tests): the gate stream such an execution applies, in execution order - boundary
 * strings as Z, X gates and a phase, then each pass's (conjugated) gates.  *n_out = records
 * written (at most cap), *n_modified = passes that would run interpreted. */
int qsv_plan_pauli_stream(const qsv_plan *plan, const qsv_pauli *paulis, int64_t n_paulis, qsv_gate *out,
                          int64_t cap, int64_t *n_out, int64_t *n_modified);

/* ---- readout (synchronous) ---- */
int qsv_norm_sq(qsv_state *st, double *out);
int qsv_prob_bit0(qsv_state *st, int k, double *out);
int qsv_collapse(qsv_state *st, int k, int outcome, double scale);
int qsv_scale(qsv_state *st, double scale);
int qsv_pmeasure(qsv_state *st, const int32_t *qubits_msb_first, int m, double *table);
int qsv_inner(qsv_state *st, const void *other_device_c128, double *re, double *im);
/* asynchronous probe table (1..4 qubits, first listed = MSB) written to DEVICE memory on the
 * state's stream: batched trajectories read their tables once at the end (noise.py:173-185 /
 * statevector.py:311-328 semantics) */
int qsv_pmeasure_async(qsv_state *st, const int32_t *qubits_msb_first, int m, double *device_table);
int qsv_max_abs_diff(qsv_state *st, const void *other_device_c128, double *out);
/* reduced density matrix of 1 or 2 qubits (first listed = MSB), row-major complex
 * 2^nq x 2^nq; branch weights ||K psi||^2 = tr(K rho K^dag) (noise.py:173-185) */
int qsv_reduced_density(qsv_state *st, int nq, const int32_t *qubits_msb_first, double *out_c128);
/* copy n_rows runs of row_len amplitudes starting at row_offsets[r] into host_out (packed,
 * row-major) with one device gather + one D2H: partial-mode recombination reads each target's
 * 2^c branch amplitudes (partition.py:182-191) */
int qsv_gather_rows(qsv_state *st, const uint64_t *row_offsets, int n_rows, uint64_t row_len, void *host_out);
/* batched noisy trajectories (run_full(prog, rng_t, noise) per trajectory, statevector.py:343-357,
 * noise.py:188-222): the state holds B = 2^batch_log2 trajectories as consecutive
 * 2^(n - batch_log2)-amplitude blocks.  In ONE pass: apply trajectory b's own dense gate on
 * gk = 0|1|2 qubits (first listed = MSB; mats = B slots of 16 complex128, the row-major
 * 2^gk x 2^gk matrix U.K_c / sqrt(p) in the first 4^gk), then reduce every trajectory's reduced
 * density of nk = 0|1|2 qubits (the next noisy gate's branch weights, or a MEASURE's p0/p1)
 * into rdm_out = B x 16 complex128 slots (host; row-major 4x4 per trajectory, the
 * 2^nk x 2^nk block top-left; returns after the copy when nk > 0) */
int qsv_noisy_batch_step(qsv_state *st, int batch_log2, int gk, const int32_t *gate_qubits_msb_first,
                         const double *mats_c128, int nk, const int32_t *next_qubits_msb_first,
                         double *rdm_out_c128);
/* the same step split in two: _async enqueues it on the state's stream (mats are staged through
 * pinned memory, so the caller may reuse them on return) and _wait blocks until it finished and
 * copies the reduced densities out (rdm_out may be NULL).  Two batched states on their own
 * streams then overlap one group's host sampling with the other group's pass. */
int qsv_noisy_batch_step_async(qsv_state *st, int batch_log2, int gk, const int32_t *gate_qubits_msb_first,
                               const double *mats_c128, int nk, const int32_t *next_qubits_msb_first);
int qsv_noisy_batch_wait(qsv_state *st, int batch_log2, double *rdm_out_c128);

#ifdef __cplusplus
}
#endif

#endif /* QSV_H */
