// Microbenchmark: HBM streaming rate of one pass's access pattern as a function of the tile's
// qubit set.  Each CTA (256 threads) reads the 2^12 amplitudes (16 B each) of one tile - the
// amplitudes whose index bits outside the tile mask equal the tile number - and writes them
// back, 16 x 128-bit accesses per thread like a r = 4 pass kernel without math.  n = 30.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tile_stream tile_stream.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cstring>
typedef unsigned long long u64;

__device__ __forceinline__ u64 deposit(u64 v, u64 mask) {
    u64 out = 0;
    for (int bit = 0; mask; ++bit) {
        const u64 low = mask & (~mask + 1);
        if ((v >> bit) & 1) out |= low;
        mask ^= low;
    }
    return out;
}

__constant__ u64 c_koff[16];
__constant__ u64 c_toff[256];
__global__ void __launch_bounds__(256, 2) k_tile(double2 *psi, u64 tmask, u64 emask) {
    // thread bits = low 8 tile bits, register bits = high 4 tile bits (offsets precomputed)
    double2 *gp = psi + deposit(blockIdx.x, emask) + c_toff[threadIdx.x];
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __ldcs(gp + c_koff[k]);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        v[k].x += 1.0;
        __stcs(gp + c_koff[k], v[k]);
    }
}
// the same with two shared-memory re-layouts (transposes of the 16 x 256 thread/register grid)
// and CTA barriers between the loads and the stores, as a 3-stage pass without math
__global__ void __launch_bounds__(256, 2) k_tile_x(double2 *psi, u64 tmask, u64 emask) {
    extern __shared__ double2 tile[];
    double2 *gp = psi + deposit(blockIdx.x, emask) + c_toff[threadIdx.x];
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __ldcs(gp + c_koff[k]);
    const unsigned t = threadIdx.x;
    for (int round = 0; round < 2; ++round) {
#pragma unroll
        for (int k = 0; k < 16; ++k) tile[(k * 256 + t) ^ (k & 7)] = v[k];
        __syncthreads();
        // thread t takes slots of 16 other threads: (t & 15) * 256 + (t >> 4) * 16 + k
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const unsigned kk = t & 15u, tt = (t >> 4) * 16u + k;
            v[k] = tile[(kk * 256 + tt) ^ (kk & 7)];
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        v[k].x += 1.0;
        __stcs(gp + c_koff[k], v[k]);
    }
}
static u64 hdeposit(u64 v, u64 mask) {
    u64 out = 0;
    for (int bit = 0; mask; ++bit) {
        const u64 low = mask & (~mask + 1);
        if ((v >> bit) & 1) out |= low;
        mask ^= low;
    }
    return out;
}

int main(int argc, char **argv) {
    const int n = 30;
    double2 *psi;
    // argv[1] = "vmm": allocate through the virtual memory management API (one physical
    // allocation, virtual range aligned to 512 MB) to see whether the driver maps it with larger
    // pages than cudaMalloc's 2 MB
    if (argc > 1 && !strcmp(argv[1], "vmm")) {
        cudaFree(0);
        CUmemAllocationProp prop = {};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = 0;
        size_t gran = 0;
        cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
        printf("recommended granularity %zu bytes\n", gran);
        const size_t bytes = sizeof(double2) << n;
        CUmemGenericAllocationHandle h;
        CUdeviceptr va = 0;
        CUresult r = cuMemCreate(&h, bytes, &prop, 0);
        if (r == CUDA_SUCCESS) r = cuMemAddressReserve(&va, bytes, (size_t)512 << 20, 0, 0);
        if (r == CUDA_SUCCESS) r = cuMemMap(va, bytes, 0, h, 0);
        CUmemAccessDesc acc = {};
        acc.location = prop.location;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (r == CUDA_SUCCESS) r = cuMemSetAccess(va, bytes, &acc, 1);
        if (r != CUDA_SUCCESS) { printf("vmm alloc failed %d\n", (int)r); return 1; }
        psi = (double2 *)va;
    } else
    if (cudaMalloc(&psi, sizeof(double2) << n) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(psi, 0, sizeof(double2) << n);
    auto mask_of = [](std::vector<int> q) { u64 m = 0; for (int x : q) m |= 1ull << x; return m; };
    struct Case { const char *name; std::vector<int> q; };
    std::vector<Case> cases = {
        {"0-11 (contiguous)", {0,1,2,3,4,5,6,7,8,9,10,11}},
        {"0-2 + 12-20", {0,1,2,12,13,14,15,16,17,18,19,20}},
        {"0-2 + 15-23", {0,1,2,15,16,17,18,19,20,21,22,23}},
        {"0-2 + 18-26", {0,1,2,18,19,20,21,22,23,24,25,26}},
        {"0-2 + 21-29 (QFT top pass)", {0,1,2,21,22,23,24,25,26,27,28,29}},
        {"0-3 + 22-29", {0,1,2,3,22,23,24,25,26,27,28,29}},
        {"0-4 + 23-29", {0,1,2,3,4,23,24,25,26,27,28,29}},
        {"0-5 + 24-29", {0,1,2,3,4,5,24,25,26,27,28,29}},
        {"0-2 + 6,12,18,19,24-28 (C2 pass 0)", {0,1,2,6,12,18,19,24,25,26,27,28}},
        {"0-2 + 10,15,16,18-22,29 (C2 pass 2)", {0,1,2,10,15,16,18,19,20,21,22,29}},
        {"0-2 + odd 11-27", {0,1,2,11,13,15,17,19,21,23,25,27}},
        {"0-2 + 9-17", {0,1,2,9,10,11,12,13,14,15,16,17}},
        {"0-2 + 5-13", {0,1,2,5,6,7,8,9,10,11,12,13}},
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto &c : cases) {
        const u64 tm = mask_of(c.q), em = ((1ull << n) - 1) & ~tm;
        u64 hi = tm, koff[16], toff[256];
        for (int i = 0; i < 8; ++i) hi &= hi - 1;
        for (int k = 0; k < 16; ++k) koff[k] = hdeposit(k, hi);
        for (int t = 0; t < 256; ++t) toff[t] = hdeposit(t, tm);
        cudaMemcpyToSymbol(c_koff, koff, sizeof(koff));
        cudaMemcpyToSymbol(c_toff, toff, sizeof(toff));
        k_tile<<<1u << (n - 12), 256>>>(psi, tm, em);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) k_tile<<<1u << (n - 12), 256>>>(psi, tm, em);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 3;
        printf("%-40s %.3f ms  %.0f GB/s", c.name, ms, 2.0 * (16.0 * (1ull << n)) / ms * 1e-6);
        cudaFuncSetAttribute(k_tile_x, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        k_tile_x<<<1u << (n - 12), 256, 65536>>>(psi, tm, em);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) k_tile_x<<<1u << (n - 12), 256, 65536>>>(psi, tm, em);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 3;
        printf("   | with 2 smem re-layouts %.3f ms  %.0f GB/s\n", ms, 2.0 * (16.0 * (1ull << n)) / ms * 1e-6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
