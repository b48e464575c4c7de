// micro_tma.cu -- microbenchmark: streaming read bandwidth of (a) the TMA
// bulk-copy ring (cp.async.bulk + mbarrier) with a trivial consumer and
// (b) a plain 128-bit LDG grid-stride loop, on the same 4 GB buffer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 micro_tma.cu -o micro_tma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     saddr(b)),
                 "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}

// mode 0: refill by warp 0 after its own consume (like stream.cuh)
// mode 1: dedicated producer warp (warp 0 does not consume)
__global__ void k_tma(const int4* v, uint64_t nvec, int chunk_bytes, int stages, int mode, unsigned long long* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk_bytes);
    uint64_t* empty = full + stages;
    const uint32_t kVec = chunk_bytes / 16;
    const uint64_t nch = (nvec + kVec - 1) / kVec;
    const int nwarps = blockDim.x / 32;
    const int consumers = mode == 1 ? nwarps - 1 : nwarps;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, consumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto chunk_of = [&](uint64_t k) { return (uint64_t)blockIdx.x + k * gridDim.x; };
    auto issue = [&](uint64_t k) {
        uint64_t c = chunk_of(k);
        if (c >= nch) return;
        int s = (int)(k % stages);
        uint64_t first = c * kVec;
        uint32_t cnt = (uint32_t)(nvec - first < kVec ? nvec - first : kVec);
        mbar_expect_tx(full + s, cnt * 16);
        bulk(sm + (size_t)s * chunk_bytes, v + first, cnt * 16, full + s);
    };
    int acc = 0;
    const int warp = threadIdx.x / 32;
    if (mode == 1 && warp == 0) {
        if (threadIdx.x == 0) {
            for (uint64_t k = 0;; ++k) {
                if (chunk_of(k) >= nch) break;
                if (k >= (uint64_t)stages) mbar_wait(empty + (k % stages), (uint32_t)(((k / stages) - 1) & 1));
                issue(k);
            }
        }
    } else {
        if (mode == 0 && threadIdx.x == 0)
            for (int s = 0; s < stages; ++s) issue(s);
        const int ctid = mode == 1 ? threadIdx.x - 32 : threadIdx.x;
        const int cthreads = consumers * 32;
        for (uint64_t k = 0;; ++k) {
            uint64_t c = chunk_of(k);
            if (c >= nch) break;
            int s = (int)(k % stages);
            mbar_wait(full + s, (uint32_t)((k / stages) & 1));
            const int4* sv = reinterpret_cast<const int4*>(sm + (size_t)s * chunk_bytes);
            uint64_t first = c * kVec;
            uint32_t cnt = (uint32_t)(nvec - first < kVec ? nvec - first : kVec);
            for (uint32_t i = ctid; i < cnt; i += cthreads) {
                int4 a = sv[i];
                acc += a.x ^ a.y ^ a.z ^ a.w;
            }
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(empty + s);
            if (mode == 0 && threadIdx.x == 0 && k >= 1) {
                uint64_t kp = k - 1;
                if (chunk_of(kp + stages) < nch) {
                    mbar_wait(empty + (kp % stages), (uint32_t)((kp / stages) & 1));
                    issue(kp + stages);
                }
            }
            __syncwarp();
        }
    }
    if (acc == 0x7fffffff) atomicAdd(out, 1ull);
}

__global__ void k_ldg(const int4* v, uint64_t nvec, unsigned long long* out) {
    int acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
        int4 a = __ldg(v + i);
        acc += a.x ^ a.y ^ a.z ^ a.w;
    }
    if (acc == 0x7fffffff) atomicAdd(out, 1ull);
}

int main() {
    const uint64_t bytes = 4ull << 30;
    int4* v;
    unsigned long long* out;
    cudaMalloc(&v, bytes);
    cudaMalloc(&out, 8);
    cudaMemset(v, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint64_t nvec = bytes / 16;
    auto timeit = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        return bytes / (best * 1e-3) / 1e9;
    };
    for (int th : {512, 1024})
        for (int per : {2, 4})
            printf("ldg   threads=%4d blocks/SM=%d : %.0f GB/s\n", th, per,
                   timeit([&] { k_ldg<<<sms * per, th>>>(v, nvec, out); }));
    for (int mode : {0, 1})
        for (int chunk : {8192, 16384, 32768})
            for (int stages : {2, 4, 6}) {
                size_t smem = (size_t)chunk * stages + 16 * stages;
                if (smem > 227 * 1024) continue;
                cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                for (int th : {256, 1024}) {
                    double gbs = timeit([&] { k_tma<<<sms, th, smem>>>(v, nvec, chunk, stages, mode, out); });
                    cudaError_t e = cudaGetLastError();
                    printf("tma mode=%d chunk=%6d stages=%d threads=%4d : %.0f GB/s %s\n", mode, chunk, stages, th, gbs,
                           e ? cudaGetErrorString(e) : "");
                }
            }
    return 0;
}
