// Host memory bandwidth of the GPU box's CPU side (what bounds the e2e
// pipelines): T threads stream-read (sum) a buffer, and stream-read +
// non-temporal-write a quarter-size output (the 16-bit pack's traffic shape).
// g++ -O3 -mavx2 -pthread tools/micro_hostbw.cpp -o tools/micro_hostbw
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
    const size_t bytes = (argc > 1 ? std::atol(argv[1]) : 8192) * (1ull << 20);
    const int T = argc > 2 ? std::atoi(argv[2]) : (int)std::thread::hardware_concurrency();
    char* a = (char*)aligned_alloc(64, bytes);
    char* b = (char*)aligned_alloc(64, bytes / 4);
    memset(a, 1, bytes);
    memset(b, 0, bytes / 4);
    std::vector<uint64_t> sums(T * 8);
    auto run = [&](int mode) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                const size_t lo = bytes / T * t / 64 * 64, hi = bytes / T * (t + 1) / 64 * 64;
                __m256i acc = _mm256_setzero_si256();
                for (size_t i = lo; i < hi; i += 64) {
                    const __m256i x = _mm256_load_si256((const __m256i*)(a + i));
                    const __m256i y = _mm256_load_si256((const __m256i*)(a + i + 32));
                    acc = _mm256_add_epi64(acc, _mm256_xor_si256(x, y));
                    if (mode == 1 && (i & 127) == 0)
                        _mm256_stream_si256((__m256i*)(b + i / 4), acc);
                }
                sums[t * 8] = (uint64_t)_mm256_extract_epi64(acc, 0);
            });
        for (auto& x : th) x.join();
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    for (int mode = 0; mode < 2; ++mode) {
        double best = 1e9;
        for (int r = 0; r < 5; ++r) best = std::min(best, run(mode));
        const double rd = bytes / best / 1e9, wr = mode ? bytes / 4 / best / 1e9 : 0;
        printf("%s, %d threads: read %.1f GB/s%s%.1f GB/s\n", mode ? "read + 1/4 NT write" : "read", T, rd,
               mode ? ", write " : "", wr);
    }
    return (int)(sums[0] & 1);
}
