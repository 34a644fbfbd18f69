// Microbenchmark: FP64 throughput of DFMA (CUDA cores), DMMA (mma.sync m8n8k4
// f64) and both interleaved, on sm_100a.  Decides whether the FP64 tensor path
// is a separate pipe worth feeding.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes fp64_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double *out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void k_dmma(double *out, double a, double b) {
    double d[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(d[i][0], d[i][1], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_both(double *out, double a, double b) {
    double x[8], d[4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma(d[i][0], d[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
float run(K kern, int blocks, int threads, double *out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<blocks, threads>>>(out, 0.999, 1e-3);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, 0.999, 1e-3);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 1 << 20);
    const int threads = 512, blocks = sms * 4;
    const double warps = (double)blocks * threads / 32;
    float t1 = run(k_dfma, blocks, threads, out);
    // DFMA: 8 chains x ITERS per thread, 2 flop each
    double f1 = (double)blocks * threads * 8 * ITERS * 2;
    float t2 = run(k_dmma, blocks, threads, out);
    // m8n8k4 per warp = 8*8*4 FMA = 256 FMA = 512 flop; 8 per iteration per warp
    double f2 = warps * 8 * ITERS * 512;
    float t3 = run(k_both, blocks, threads, out);
    double f3 = (double)blocks * threads * 8 * ITERS * 2 + warps * 4 * ITERS * 512;
    printf("{\"sms\": %d, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"both_tflops\": %.2f, "
           "\"dfma_ms\": %.3f, \"dmma_ms\": %.3f, \"both_ms\": %.3f}\n",
           sms, f1 / t1 / 1e9, f2 / t2 / 1e9, f3 / t3 / 1e9, t1, t2, t3);
    return 0;
}
