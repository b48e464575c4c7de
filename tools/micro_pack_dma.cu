// Host pack + H2D probe for the packed pipeline: T host threads, each packs
// pieces of P points from a pinned int32 (x,y) source into its own small
// pinned staging ring (regular or non-temporal stores) and DMAs each piece
// to the device on its own stream.  Reports points/s for n = 1e8.
// nvcc -O3 -std=c++17 -Xcompiler -mavx2,-pthread tools/micro_pack_dma.cu -o tools/micro_pack_dma
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>

static void pack(const int32_t* src, uint32_t* dst, uint64_t m, bool nt) {
    const __m256i perm = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7), one = _mm256_set1_epi32(1);
    for (uint64_t i = 0; i + 8 <= m; i += 8) {
        const __m256i a = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i*)(src + 2 * i)), perm);
        const __m256i b = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i*)(src + 2 * i + 8)), perm);
        const __m256i s = _mm256_sub_epi32(_mm256_permute2x128_si256(a, b, 0x20), one);
        const __m256i y = _mm256_sub_epi32(_mm256_permute2x128_si256(a, b, 0x31), one);
        const __m256i w = _mm256_or_si256(s, _mm256_slli_epi32(y, 16));
        if (nt) _mm256_stream_si256((__m256i*)(dst + i), w);
        else _mm256_store_si256((__m256i*)(dst + i), w);
    }
    if (nt) _mm_sfence();
}

int main() {
    const uint64_t n = 100'000'000;
    int32_t* src;
    cudaMallocHost(&src, n * 8);
    for (uint64_t i = 0; i < 2 * n; ++i) src[i] = 1 + (int32_t)((i * 2654435761u) & 0xFFFF);
    uint32_t* dev;
    cudaMalloc(&dev, n * 4);
    const int TMAX = 16;
    const uint64_t PMAX = 1048576;
    cudaStream_t st[TMAX];
    uint32_t* ring[TMAX][3];
    cudaEvent_t ev[TMAX][3];
    for (int t = 0; t < TMAX; ++t) {
        cudaStreamCreateWithFlags(&st[t], cudaStreamNonBlocking);
        for (int k = 0; k < 3; ++k) {
            cudaMallocHost(&ring[t][k], PMAX * 4);
            cudaEventCreateWithFlags(&ev[t][k], cudaEventDisableTiming);
        }
    }
    for (int nt : {1, 0})
        for (uint64_t P : {65536ull, 262144ull, 1048576ull})
            for (int T : {8, 16}) {
                double best = 1e9;
                for (int rep = 0; rep < 3; ++rep) {
                    for (int t = 0; t < T; ++t)
                        for (int k = 0; k < 3; ++k) cudaEventRecord(ev[t][k], st[t]);
                    cudaDeviceSynchronize();
                    std::atomic<uint64_t> next{0};
                    auto t0 = std::chrono::steady_clock::now();
                    std::vector<std::thread> th;
                    for (int t = 0; t < T; ++t)
                        th.emplace_back([&, t] {
                            for (uint64_t it = 0;; ++it) {
                                const uint64_t off = next.fetch_add(P);
                                if (off >= n) break;
                                const uint64_t m = std::min(P, n - off);
                                const int k = (int)(it % 3);
                                cudaEventSynchronize(ev[t][k]);
                                pack(src + 2 * off, ring[t][k], m, nt);
                                cudaMemcpyAsync(dev + off, ring[t][k], m * 4, cudaMemcpyHostToDevice, st[t]);
                                cudaEventRecord(ev[t][k], st[t]);
                            }
                            cudaStreamSynchronize(st[t]);
                        });
                    for (auto& x : th) x.join();
                    best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
                }
                printf("%s piece=%7llu T=%2d: %.2f Gpts/s\n", nt ? "NT    " : "cached", (unsigned long long)P, T,
                       n / best / 1e9);
            }
    return 0;
}
