// micro_dsmem.cu -- random 16-bit lookups into a table distributed over a
// thread-block cluster (DSMEM), vs the same lookups into the CTA's own smem.
// Reports lookups per cycle per SM.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 micro_dsmem.cu -o micro_dsmem
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

template <int CL, bool REMOTE>
__global__ void k(uint32_t iters, unsigned long long* out) {
    extern __shared__ uint16_t T[];
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t words = 64 * 1024;  // 128 KB per CTA
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) T[i] = (uint16_t)i;
    cl.sync();
    uint32_t x = (blockIdx.x * 1315423911u) ^ (threadIdx.x * 2654435761u);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        uint16_t v[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
            x = x * 1664525u + 1013904223u;
            const uint32_t col = x >> 12;  // 20-bit column
            if (REMOTE) {
                const uint16_t* p = cl.map_shared_rank(T, (col >> 16) % CL);
                v[k2] = p[col & 0xFFFF];
            } else {
                v[k2] = T[col & 0xFFFF];
            }
        }
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) acc += v[k2];
    }
    cl.sync();
    if (acc == 0x12345678) atomicAdd(out, 1ull);
}

template <int CL, bool REMOTE>
void run(int sms, unsigned long long* out) {
    auto fn = k<CL, REMOTE>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    if (CL > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    int grid = (sms / CL) * CL;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = 128 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint32_t iters = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, fn, iters, out);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, fn, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double lookups = (double)grid * 1024 * iters * 8;
    printf("cluster=%2d remote=%d grid=%d: %.3f ms, %.2f G lookups/s, %.2f lookups/cycle/SM %s\n", CL, REMOTE, grid, ms,
           lookups / ms / 1e6, lookups / (ms * 1e-3) / (clk * 1e3) / grid, e ? cudaGetErrorString(e) : "");
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out;
    cudaMalloc(&out, 8);
    run<1, false>(sms, out);
    run<2, true>(sms, out);
    run<4, true>(sms, out);
    run<8, true>(sms, out);
    run<16, true>(sms, out);
    return 0;
}
