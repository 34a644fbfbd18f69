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
std::string jit_source(const Plan &P, int pass, bool host = false);

// Compiles (or fetches from the cache) every pass kernel of P for `device`;
// fills P.jit_funcs.  Returns QSV_OK or an error status with `err` set.
int jit_prepare(Plan &P, int device, std::string &err);

// Compiles one source to a cubin for sm_100a (no GPU needed).  Returns the
// NVRTC log in `log`; empty cubin on failure.
std::string jit_compile_cubin(const std::string &src, std::string &log);

// Launches pass `pass` of a prepared plan.
int jit_launch(const Plan &P, int pass, void *psi, int n, cudaStream_t stream, std::string &err);

}  // namespace qsv
