// Host pack-rate probe for the packed pipeline (same loop as abi.cu pack16):
// points/s vs thread count, SSE2 vs AVX2, from a large (pinned-like) buffer.
// g++ -O3 -std=c++17 -pthread tools/micro_pack.cpp -o tools/micro_pack
#include <immintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static uint32_t pack_sse2(const int32_t* src, uint32_t* dst, uint64_t m, uint32_t base, uint32_t wcheck,
                          uint32_t qmax) {
    const __m128i vbase = _mm_set1_epi32((int)base), vone = _mm_set1_epi32(1);
    const __m128i sign = _mm_set1_epi32((int)0x80000000u);
    const __m128i wlim = _mm_set1_epi32((int)(wcheck ^ 0x80000000u)), qlim = _mm_set1_epi32((int)(qmax ^ 0x80000000u));
    __m128i okv = _mm_set1_epi32(-1);
    for (uint64_t i = 0; i + 4 <= m; i += 4) {
        const __m128i a = _mm_loadu_si128((const __m128i*)(src + 2 * i));
        const __m128i b = _mm_loadu_si128((const __m128i*)(src + 2 * i + 4));
        const __m128i a2 = _mm_shuffle_epi32(a, _MM_SHUFFLE(3, 1, 2, 0));
        const __m128i b2 = _mm_shuffle_epi32(b, _MM_SHUFFLE(3, 1, 2, 0));
        const __m128i s = _mm_sub_epi32(_mm_unpacklo_epi64(a2, b2), vbase);
        const __m128i ym1 = _mm_sub_epi32(_mm_unpackhi_epi64(a2, b2), vone);
        okv = _mm_and_si128(okv, _mm_cmplt_epi32(_mm_xor_si128(s, sign), wlim));
        okv = _mm_and_si128(okv, _mm_cmplt_epi32(_mm_xor_si128(ym1, sign), qlim));
        _mm_stream_si128((__m128i*)(dst + i), _mm_or_si128(s, _mm_slli_epi32(ym1, 16)));
    }
    _mm_sfence();
    return (uint32_t)(_mm_movemask_epi8(okv) != 0xFFFF);
}

__attribute__((target("avx2"))) static uint32_t pack_avx2(const int32_t* src, uint32_t* dst, uint64_t m,
                                                          uint32_t base, uint32_t wcheck, uint32_t qmax) {
    const __m256i vbase = _mm256_set1_epi32((int)base), vone = _mm256_set1_epi32(1);
    const __m256i wl = _mm256_set1_epi32((int)wcheck), ql = _mm256_set1_epi32((int)qmax);
    const __m256i perm = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
    __m256i bad = _mm256_setzero_si256();
    for (uint64_t i = 0; i + 8 <= m; i += 8) {
        const __m256i a = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i*)(src + 2 * i)), perm);
        const __m256i b = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i*)(src + 2 * i + 8)), perm);
        const __m256i xs = _mm256_permute2x128_si256(a, b, 0x20), ys = _mm256_permute2x128_si256(a, b, 0x31);
        const __m256i s = _mm256_sub_epi32(xs, vbase), ym1 = _mm256_sub_epi32(ys, vone);
        // unsigned v >= lim  <=>  max(v, lim) == v
        bad = _mm256_or_si256(bad, _mm256_cmpeq_epi32(_mm256_max_epu32(s, wl), s));
        bad = _mm256_or_si256(bad, _mm256_cmpeq_epi32(_mm256_max_epu32(ym1, ql), ym1));
        _mm256_stream_si256((__m256i*)(dst + i), _mm256_or_si256(s, _mm256_slli_epi32(ym1, 16)));
    }
    _mm_sfence();
    return (uint32_t)!_mm256_testz_si256(bad, bad);
}


// 42-bit packing (abi.cu pack42_any, int32 input): scalar, and an AVX2 form
// (4 points per 256-bit vector, 12 points -> 4 words of 3).
static uint32_t pack42_scalar(const int32_t* src, uint64_t* dst, uint64_t m, uint32_t base, uint32_t ybase,
                              uint32_t wcheck, uint32_t qmax) {
    uint32_t bad = 0;
    auto val = [&](uint64_t k) -> uint64_t {
        const uint64_t s = (uint32_t)src[2 * k] - base, t = (uint32_t)src[2 * k + 1] - ybase;
        bad |= (uint32_t)(s >= wcheck) | (uint32_t)(t >= qmax);
        return (s & 0x1FFFFF) | ((t & 0x1FFFFF) << 21);
    };
    for (uint64_t w = 0; w < m / 3; ++w) {
        const uint64_t v0 = val(3 * w), v1 = val(3 * w + 1), v2 = val(3 * w + 2);
        _mm_stream_si128((__m128i*)(dst + 2 * w), _mm_set_epi64x((long long)((v1 >> 22) | (v2 << 20)),
                                                                  (long long)(v0 | (v1 << 42))));
    }
    _mm_sfence();
    return bad;
}

__attribute__((target("avx2"))) static uint32_t pack42_avx2(const int32_t* src, uint64_t* dst, uint64_t m,
                                                            uint32_t base, uint32_t ybase, uint32_t wcheck,
                                                            uint32_t qmax) {
    const __m256i sub = _mm256_setr_epi32((int)base, (int)ybase, (int)base, (int)ybase, (int)base, (int)ybase,
                                          (int)base, (int)ybase);
    const __m256i lim = _mm256_setr_epi32((int)wcheck, (int)qmax, (int)wcheck, (int)qmax, (int)wcheck, (int)qmax,
                                          (int)wcheck, (int)qmax);
    const __m256i m21 = _mm256_set1_epi64x(0x1FFFFF);
    __m256i badv = _mm256_setzero_si256();
    alignas(32) uint64_t v[12];
    uint64_t w = 0;
    for (uint64_t i = 0; i + 12 <= m; i += 12, w += 4) {
#pragma GCC unroll 3
        for (int j = 0; j < 3; ++j) {
            const __m256i d = _mm256_sub_epi32(_mm256_loadu_si256((const __m256i*)(src + 2 * i + 8 * j)), sub);
            badv = _mm256_or_si256(badv, _mm256_cmpeq_epi32(_mm256_max_epu32(d, lim), d));
            const __m256i q = _mm256_or_si256(_mm256_and_si256(d, m21), _mm256_slli_epi64(_mm256_srli_epi64(d, 32), 21));
            _mm256_store_si256((__m256i*)(v + 4 * j), q);
        }
        uint64_t o[8];
#pragma GCC unroll 4
        for (int g = 0; g < 4; ++g) {
            const uint64_t a = v[3 * g], b = v[3 * g + 1], c = v[3 * g + 2];
            o[2 * g] = a | (b << 42);
            o[2 * g + 1] = (b >> 22) | (c << 20);
        }
        _mm256_stream_si256((__m256i*)(dst + 2 * w), _mm256_loadu_si256((const __m256i*)o));
        _mm256_stream_si256((__m256i*)(dst + 2 * w + 4), _mm256_loadu_si256((const __m256i*)(o + 4)));
    }
    _mm_sfence();
    return (uint32_t)!_mm256_testz_si256(badv, badv);
}

static int main42() {
    const uint64_t n = 100'000'008;  // a multiple of 12
    std::vector<int32_t> src(2 * n);
    for (uint64_t i = 0; i < 2 * n; ++i) src[i] = 1 + (int32_t)((i * 2654435761u) & 0xFFFFF);
    uint64_t* d1 = (uint64_t*)aligned_alloc(64, (n / 3 + 8) * 16);
    uint64_t* d2 = (uint64_t*)aligned_alloc(64, (n / 3 + 8) * 16);
    memset(d1, 0, (n / 3 + 8) * 16);
    memset(d2, 0, (n / 3 + 8) * 16);
    // correctness of the AVX2 form against the scalar one
    pack42_scalar(src.data(), d1, 1200000, 1, 1, 1 << 20, 1 << 20);
    pack42_avx2(src.data(), d2, 1200000, 1, 1, 1 << 20, 1 << 20);
    printf("pack42 avx2 == scalar: %s\n", memcmp(d1, d2, 800000 * 8) == 0 ? "yes" : "NO");
    for (int avx : {0, 1})
        for (int T : {1, 4, 8, 16}) {
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> th;
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&, t] {
                        const uint64_t lo = (n * t / T) / 12 * 12, hi = t + 1 == T ? n : (n * (t + 1) / T) / 12 * 12;
                        if (avx) pack42_avx2(src.data() + 2 * lo, d2 + 2 * (lo / 3), hi - lo, 1, 1, 1 << 20, 1 << 20);
                        else pack42_scalar(src.data() + 2 * lo, d1 + 2 * (lo / 3), hi - lo, 1, 1, 1 << 20, 1 << 20);
                    });
                for (auto& x : th) x.join();
                best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            }
            printf("pack42 %s T=%2d: %.2f Gpts/s\n", avx ? "avx2  " : "scalar", T, n / best / 1e9);
        }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && !strcmp(argv[1], "42")) return main42();
    const uint64_t n = 100'000'000;
    std::vector<int32_t> src(2 * n);
    for (uint64_t i = 0; i < 2 * n; ++i) src[i] = 1 + (int32_t)((i * 2654435761u) & 0xFFFF);
    uint32_t* dst = (uint32_t*)aligned_alloc(64, n * 4);
    memset(dst, 0, n * 4);
    for (int avx : {0, 1})
        for (int T : {1, 2, 4, 8, 16}) {
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> th;
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&, t] {
                        const uint64_t lo = (n * t / T) & ~7ull, hi = t + 1 == T ? n : (n * (t + 1) / T) & ~7ull;
                        if (avx) pack_avx2(src.data() + 2 * lo, dst + lo, hi - lo, 1, 65536, 65536);
                        else pack_sse2(src.data() + 2 * lo, dst + lo, hi - lo, 1, 65536, 65536);
                    });
                for (auto& x : th) x.join();
                best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            }
            printf("%s T=%2d: %.2f Gpts/s (%.0f GB/s read+write)\n", avx ? "avx2" : "sse2", T, n / best / 1e9,
                   n * 12.0 / best / 1e9);
        }
    return 0;
}
