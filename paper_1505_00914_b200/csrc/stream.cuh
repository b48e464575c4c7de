// stream.cuh -- TMA bulk staging of the point stream into a shared-memory
// ring (cp.async.bulk global->shared with mbarrier completion; SASS UBLKCP).
//
// The reduction kernels are HBM-bound only if enough bytes are in flight per
// SM.  With 1024 threads at 64 registers the register file is full, so
// register double-buffering caps in-flight data near 64 KB/SM; the ring moves
// it into shared memory instead.  Warp 0 is a dedicated producer (one elected
// lane issues one bulk copy per stage and refills a stage as soon as all
// consumer warps have released it); warps 1..31 consume.  Measured on B200
// (tools/micro_tma.cu, trivial consumer, 4 GB): producer warp + 4 x 32 KB
// stages 7.32 TB/s vs 6.87 TB/s for the best plain 128-bit LDG loop and
// 5.8 TB/s when a consumer warp also refills.
//
// A chunk holds exactly 2 x 16-byte vectors per consumer thread (31 warps x
// 32 x 2 x 16 B = 31,744 B = 3,968 points); CTA b walks chunks b, b+grid, ...
#pragma once
#include <cstdint>

namespace chpstream {

constexpr int kConsumerWarps = 31;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kChunkVec = kConsumers * 2;    // 16-byte vectors per chunk
constexpr int kChunkBytes = kChunkVec * 16;  // 31,744 B

__device__ __forceinline__ uint32_t saddr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(saddr(bar)),
        "r"(parity)
        : "memory");
}
// 1D bulk copy global -> shared, completion counted in bytes on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}

// Shared-memory layout: [ring: stages x kChunkBytes][full: stages][empty: stages]
struct Ring {
    uint8_t* buf;
    uint64_t* full;
    uint64_t* empty;
    int stages;
};

__device__ __forceinline__ Ring ring_at(uint8_t* base, int stages) {
    Ring r;
    r.buf = base;
    r.full = reinterpret_cast<uint64_t*>(base + (size_t)stages * kChunkBytes);
    r.empty = r.full + stages;
    r.stages = stages;
    return r;
}

__host__ __device__ constexpr size_t ring_bytes(int stages) {
    return (size_t)stages * kChunkBytes + 2 * 8 * (size_t)stages;
}

// Streams the 16-byte vectors v[0..nvec) through the ring.  Consumer thread
// c (warps 1..31) receives vectors (c, c + kConsumers) of every full chunk
// as g(a, b); vectors of a final partial chunk go one at a time to g1(a).
// Requires blockDim.x == 1024; called by all threads; ends with a barrier.
// Returns false on the producer warp (which consumed nothing).
template <typename G, typename G1>
__device__ __forceinline__ void tma_stream(const int4* __restrict__ v, uint64_t nvec, Ring r, G&& g, G1&& g1) {
    const uint64_t nchunks = (nvec + kChunkVec - 1) / kChunkVec;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < r.stages; ++s) {
            mbar_init(r.full + s, 1);
            mbar_init(r.empty + s, kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto chunk_of = [&](uint64_t k) { return (uint64_t)blockIdx.x + k * gridDim.x; };
    if (tid < 32) {
        if (tid == 0) {  // producer
            for (uint64_t k = 0;; ++k) {
                const uint64_t c = chunk_of(k);
                if (c >= nchunks) break;
                const int s = (int)(k % r.stages);
                if (k >= (uint64_t)r.stages) mbar_wait(r.empty + s, (uint32_t)(((k / r.stages) - 1) & 1));
                const uint64_t first = c * kChunkVec;
                const uint32_t cnt = (uint32_t)(nvec - first < kChunkVec ? nvec - first : kChunkVec);
                mbar_expect_tx(r.full + s, cnt * 16);
                bulk_load(r.buf + (size_t)s * kChunkBytes, v + first, cnt * 16, r.full + s);
            }
        }
    } else {
        const uint32_t ct = tid - 32;
        for (uint64_t k = 0;; ++k) {
            const uint64_t c = chunk_of(k);
            if (c >= nchunks) break;
            const int s = (int)(k % r.stages);
            mbar_wait(r.full + s, (uint32_t)((k / r.stages) & 1));
            const int4* sv = reinterpret_cast<const int4*>(r.buf + (size_t)s * kChunkBytes);
            const uint64_t first = c * kChunkVec;
            const uint32_t cnt = (uint32_t)(nvec - first < kChunkVec ? nvec - first : kChunkVec);
            if (cnt == (uint32_t)kChunkVec) {
                g(sv[ct], sv[ct + kConsumers]);
            } else {
                for (uint32_t i = ct; i < cnt; i += kConsumers) g1(sv[i]);
            }
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(r.empty + s);
        }
    }
    __syncthreads();
}

}  // namespace chpstream
