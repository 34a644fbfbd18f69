// Sustained FP64 rate under the board's power cap: back-to-back DADD / DFMA kernels for a few
// seconds on every SM (16 warps/SM, 16 independent chains per thread), the rate reported per
// 0.25 s window.  Run with `nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active
// --format=csv -lms 200` beside it: a burst measurement (fp64_pipes.cu, ~1 ms) sees the full
// 1965 MHz clock, a 50 ms state-vector step does not.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_sustained fp64_sustained.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1 << 15;

template <int FMA>
__global__ void __launch_bounds__(256) k(double *out, double c) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (FMA) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(x[i]) : "d"(c));
            else asm volatile("add.f64 %0, %0, %1;" : "+d"(x[i]) : "d"(c));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int FMA>
void run(const char *name, int sms, double *out, double seconds) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 2 * sms;
    const double per_launch = (double)grid * 256 * ITERS * 16;
    double total = 0;
    while (total < seconds) {
        cudaEventRecord(e0);
        int launches = 0;
        for (; launches < 8; ++launches) k<FMA><<<grid, 256>>>(out, 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        total += ms * 1e-3;
        printf("%s t=%.2fs  %.2f T lane-instr/s\n", name, total, launches * per_launch / ms * 1e-9);
    }
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double *out;
    cudaMalloc(&out, 4096);
    run<0>("DADD", p.multiProcessorCount, out, 4.0);
    run<1>("DFMA", p.multiProcessorCount, out, 4.0);
    return 0;
}
