// Per-pass kernel specialisation (runtime code generation + NVRTC, sm_100a).
//
// The interpreted pass kernel (qsv_kernels.cuh) decodes every op per thread
// and tests register positions / factors at run time; the profile showed that
// decode and dispatch cost more instructions than the FP64 math itself.  For
// large states the launcher instead emits straight-line CUDA for each pass in
// which register positions, smem offsets, matrices and control classes are
// compile-time constants, compiles it with NVRTC for sm_100a and launches it
// through the driver API.  Kernels are cached by source text, so a plan that
// is executed repeatedly (bench steps, trajectories, repeated run_full calls)
// compiles once per process.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "qsv_plan.h"

namespace qsv {

// true when libnvrtc + libcuda could be loaded; `why` explains a failure
bool jit_available(std::string &why);

// CUDA source of the specialised kernel for pass `pass` of plan P (extern "C"
// entry point `qsv_pass`).  Pure host code (testable without a GPU).
std::string jit_source(const Plan &P, int pass, bool host = false, double *fp64_per_amp = nullptr,
                       uint64_t xmask = 0, const std::vector<int> *probe = nullptr);

// Probe-out variant of pass `pass`: the |amp|^2 of its outputs accumulated per key
// over `probe` (first = MSB) into per-CTA partials probe_out[grid][2^|probe|]; the
// launch uses exactly `grid` CTAs (the caller sizes the partials and the finish).
int jit_probe_prepare(const Plan &P, int pass, const std::vector<int> &probe, int device, void **fn, int *grid,
                      std::string &err);
int jit_launch_probe(const Plan &P, int pass, void *fn, int grid, void *psi, int n, cudaStream_t stream,
                     std::string &err, unsigned long long basis, double *probe_out);

// Exchange-out variant of pass `pass` (xmask = exchanged positions, all tile-base
// bits of that pass): stores go to dst8[bits at xmask] + (index with those bits
// replaced by self_bits).  Compiled on demand and cached like the pass kernels.
int jit_exchange_prepare(const Plan &P, int pass, uint64_t xmask, int device, void **fn, int *grid, std::string &err);
int jit_launch_exchange(const Plan &P, int pass, void *fn, int grid_cap, void *psi, int n, cudaStream_t stream,
                        std::string &err, unsigned long long basis, const unsigned long long *dst8,
                        unsigned long long self_bits);

// Cost model: decides for every super-pass whether its inner passes run as one
// L2-resident persistent kernel (one HBM pass) or as flat passes (one HBM pass
// each), from the FP64 work the generator emits per amplitude.  Fills
// P.super_use.  `sms` = multiprocessor count.
void jit_choose_supers(Plan &P, int sms);

// Compiles (or fetches from the cache) every pass kernel of P for `device`;
// fills P.jit_funcs.  Returns QSV_OK or an error status with `err` set.
int jit_prepare(Plan &P, int device, std::string &err);

// Compiles one source to a cubin for sm_100a (no GPU needed).  Returns the
// NVRTC log in `log`; empty cubin on failure.
std::string jit_compile_cubin(const std::string &src, std::string &log);

// Source of the persistent kernel of super-pass `si` (all its inner passes on
// L2-resident super-tiles, grid barrier between inner passes).
std::string jit_super_source(const Plan &P, int si, bool host = false);

// log2 of the number of super-tiles processed together (L2 budget ~64 MB)
int super_batch(const Plan &P);

// cp.async double buffering of tiles in the generated kernels (QSV_JIT_DBUF)
bool jit_double_buffer();

// true when the plan's super-passes run as L2-resident persistent kernels
bool use_supers(const Plan &P);

// build_plan with the register qubits chosen per pass (r = 4 where it does not
// add FP64 work, else r = 5) when auto_r and r = 5 (see qsv_jit.cpp)
Plan build_plan_auto(const std::vector<GateRec> &recs, int n, int m, int r, int L, int s, bool auto_r);

// The uniform scale every pass's specialised kernel expects the stored state
// to carry (stored = true / scale); entry passes.size() is the plan's output (1).
const std::vector<double> &pass_scales(const Plan &P);

// Launches pass `pass` of a prepared plan over the whole state.  `basis` !=
// ~0 means the state is the basis state |basis> and is not read (single-buffer
// kernels synthesise the tiles; see jit_basis_fusable).
int jit_launch(const Plan &P, int pass, void *psi, int n, cudaStream_t stream, std::string &err,
               unsigned long long basis = ~0ull, const void *ptab = nullptr);

// build_plan_auto, or with `product` a product-start plan (Plan::product) when the
// stream has leading single-qubit gates to absorb
Plan build_plan_start(const std::vector<GateRec> &recs, int n, int m, int r, int L, int s, bool auto_r,
                      bool product);

// Cold calls (a plan whose kernels are not compiled yet): jit_start_async queues
// every missing pass kernel on a background NVRTC pool and returns at once;
// jit_try_pass loads pass `pass` if its kernel has finished compiling (*ready);
// jit_launch_partial launches such a loaded pass.  Once every pass is loaded
// the plan is an ordinary prepared plan (jit_ready).  Flat plans only.
bool jit_ready(const Plan &P, int device);
void jit_wait_async();  // blocks until no background compile is queued or running
int jit_start_async(Plan &P, int device, std::string &err);
int jit_try_pass(Plan &P, int pass, int device, bool *ready, std::string &err);
int jit_launch_partial(const Plan &P, int pass, void *psi, int n, cudaStream_t stream, std::string &err,
                       unsigned long long basis, const void *ptab);

// register qubits (k = 0..R-1) of pass 0's first stage: the `regs` of product_tables
std::vector<int> product_regs(const Plan &P);

// Launches the persistent kernel of super-pass `si` (needs a 4-byte device
// counter for the grid barrier).
int jit_launch_super(const Plan &P, int si, void *psi, unsigned *bar, cudaStream_t stream, std::string &err);

}  // namespace qsv
