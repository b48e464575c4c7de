// abi.cu -- context management and the host-buffer pipelines of the C ABI.
//
// chp_pipeline_host is what the C++ drop-in (reducer::reduce,
// build_polyline, hulls::melkman) and the end-to-end bench call: the input
// is streamed to the device in chunks on a copy stream while K1 reduces the
// previous chunk on the compute stream (two device buffers, event-ordered),
// then K3 (+K4) run on device and only L / the chain / the hull come back.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <immintrin.h>
#include <mutex>
#include <thread>
#include <vector>

#include "chp_internal.cuh"

namespace {

// Persistent host workers for the packed pipeline: run(f, k) calls f(i) for
// i in [0, k) on the workers and the caller, and returns when all are done.
// One job at a time (the pipeline is single-threaded per context).  Only the
// k - 1 workers a job uses are waited for, and a worker spins briefly on the
// job counter before sleeping, so back-to-back calls (a chunk loop, or a
// caller timing 0.2-1 ms calls) do not pay a futex wake-up per worker.
class HostPool {
  public:
    explicit HostPool(int workers) {
        for (int i = 0; i < workers; ++i) th_.emplace_back([this, i] { loop(i + 1); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_.store(true);
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int parts() const { return (int)th_.size() + 1; }
    // Parts worth waking for m items (>= 32 Ki each): small host calls stay
    // on the caller's thread.
    int parts_for(uint64_t m) const {
        const uint64_t k = (m + (32u << 10) - 1) / (32u << 10);
        return (int)std::max<uint64_t>(1, std::min<uint64_t>(k, (uint64_t)parts()));
    }
    // f(i) for i in [0, k) (k = parts() by default).
    void run(const std::function<void(int)>& f, int k = 0) {
        if (k <= 0 || k > parts()) k = parts();
        if (k == 1) {
            f(0);
            return;
        }
        job_ = &f;
        pending_.store(k - 1);
        {
            // generation and part count in one word, so a worker that wakes
            // late never pairs one job's generation with another's count
            std::lock_guard<std::mutex> g(m_);
            const uint64_t gen = (gen_.load(std::memory_order_relaxed) >> 8) + 1;
            gen_.store((gen << 8) | (uint64_t)k, std::memory_order_release);
        }
        cv_.notify_all();
        f(0);
        const auto t0 = std::chrono::steady_clock::now();
        while (pending_.load(std::memory_order_acquire) != 0) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) {
                std::unique_lock<std::mutex> lk(m_);
                done_.wait(lk, [this] { return pending_.load() == 0; });
                break;
            }
            _mm_pause();
        }
        job_ = nullptr;
    }

  private:
    void loop(int id) {
        uint64_t seen = 0;
        for (;;) {
            // Spin up to ~0.5 ms for the next job, then sleep.
            const auto t0 = std::chrono::steady_clock::now();
            while (gen_.load(std::memory_order_acquire) == seen && !stop_.load(std::memory_order_relaxed) &&
                   std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(500))
                _mm_pause();
            if (gen_.load(std::memory_order_acquire) == seen) {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_.load() || gen_.load() != seen; });
            }
            if (stop_.load()) return;
            seen = gen_.load(std::memory_order_acquire);
            if (id >= (int)(seen & 0xFF)) continue;  // not part of this job
            (*job_)(id);
            if (pending_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
                std::lock_guard<std::mutex> g(m_);
                done_.notify_one();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    std::atomic<uint64_t> gen_{0};  // (generation << 8) | parts of the current job
    std::atomic<int> pending_{0};
    std::atomic<bool> stop_{false};
};

HostPool* pool_of(chp_ctx* ctx) {
    if (!ctx->pool) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        int parts = ctx->pool_parts > 0 ? ctx->pool_parts : (int)std::min(hw, 32u);
        // CHP_HOST_THREADS: the caller's share of the host (e.g. one process
        // per GPU on a multi-GPU box: cores / local ranks; bench.py sets it)
        if (const char* e = std::getenv("CHP_HOST_THREADS"))
            if (std::atoi(e) > 0) parts = std::min(std::atoi(e), 64);
        ctx->pool = new HostPool(std::max(parts, 1) - 1);
    }
    return static_cast<HostPool*>(ctx->pool);
}

constexpr uint64_t kChunkPts = 16ull << 20;  // 16 Mi points = 128 MiB per chunk

void free_buf(DevBuf& b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// A host point array: int32 pairs (the C ABI) or int64 pairs (the
// reference's Point, read directly by the C++ drop-in, optionally with the
// axes swapped).  Only an int32 array can be DMA'd as is.
struct HostPts {
    const int32_t* p32 = nullptr;
    const int64_t* p64 = nullptr;
    bool swap = false;  // p64 only: read (y, x)
    int64_t x(uint64_t i) const { return p64 ? p64[2 * i + (swap ? 1 : 0)] : p32[2 * i]; }
    int64_t y(uint64_t i) const { return p64 ? p64[2 * i + (swap ? 0 : 1)] : p32[2 * i + 1]; }
    bool pinned32() const { return p32 && is_pinned(p32); }
};

// Points [off, off+m) into int32 pairs at dst (pinned staging) on the host
// pool: a copy for int32 input, a checked narrowing for int64 input.
// Returns nonzero if a coordinate does not fit int32.
uint32_t stage_copy(chp_ctx* ctx, const HostPts& in, uint64_t off, uint64_t m, int32_t* dst) {
    HostPool* pool = pool_of(ctx);
    const int parts = pool->parts_for(m);
    std::vector<uint32_t> bad((size_t)parts, 0u);
    pool->run([&](int i) {
        const uint64_t lo = m * (uint64_t)i / parts, hi = m * (uint64_t)(i + 1) / parts;
        if (in.p32) {
            std::memcpy(dst + 2 * lo, in.p32 + 2 * (off + lo), (size_t)(hi - lo) * 8);
            return;
        }
        uint32_t b = 0;
        for (uint64_t k = lo; k < hi; ++k) {
            const int64_t x = in.x(off + k), y = in.y(off + k);
            b |= (uint32_t)(x != (int32_t)x) | (uint32_t)(y != (int32_t)y);
            dst[2 * k] = (int32_t)x;
            dst[2 * k + 1] = (int32_t)y;
        }
        bad[(size_t)i] = b;
    }, parts);
    uint32_t any = 0;
    for (uint32_t b : bad) any |= b;
    return any;
}

// Streams h_xy[0..n) to the device in chunks and enqueues launch(d, m) on
// the compute stream for each chunk as soon as its copy has landed.  With
// d_dest the chunks land in d_dest[0..2n) (the input stays resident), else
// in two alternating device staging buffers.
template <typename Launch>
int stream_chunks(chp_ctx* ctx, const HostPts& in, uint64_t n, Launch&& launch, int32_t* d_dest = nullptr,
                  uint32_t* narrow_bad = nullptr) {
    if (n == 0) return CHP_OK;
    const bool pinned = in.pinned32();
    const uint64_t chunk = std::min<uint64_t>(kChunkPts, n);
    const size_t bytes = (size_t)chunk * 8;
    int rc;
    for (int b = 0; b < 2 && !d_dest; ++b)
        if ((rc = chp_ensure(ctx, ctx->stage_dev[b], bytes))) return rc;
    if (!pinned && ctx->stage_bytes < bytes) {
        for (int b = 0; b < 2; ++b) {
            if (ctx->stage_host[b]) cudaFreeHost(ctx->stage_host[b]);
            ctx->stage_host[b] = nullptr;
        }
        for (int b = 0; b < 2; ++b) CHP_CUDA(ctx, cudaMallocHost(&ctx->stage_host[b], bytes));
        ctx->stage_bytes = bytes;
    }
    // The previous call may still be reading the staging buffers.
    for (int b = 0; b < 2; ++b) {
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
    }
    uint64_t k = 0;
    for (uint64_t off = 0; off < n; off += chunk, ++k) {
        const int b = (int)(k & 1);
        const uint64_t m = std::min<uint64_t>(chunk, n - off);
        const int32_t* src = in.p32 ? in.p32 + 2 * off : nullptr;
        if (!pinned) {
            // The previous H2D out of this staging buffer must have finished.
            // The copy (or int64 narrowing) into pinned staging runs on the
            // host pool (one thread copies ~14 GB/s, a quarter of what PCIe
            // drains).
            CHP_CUDA(ctx, cudaEventSynchronize(ctx->ev_copied[b]));
            const uint32_t nb = stage_copy(ctx, in, off, m, static_cast<int32_t*>(ctx->stage_host[b]));
            if (narrow_bad) *narrow_bad |= nb;
            src = (const int32_t*)ctx->stage_host[b];
        }
        int32_t* dst = d_dest ? d_dest + 2 * off : (int32_t*)ctx->stage_dev[b].p;
        CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_consumed[b], 0));
        CHP_CUDA(ctx, cudaMemcpyAsync(dst, src, (size_t)m * 8, cudaMemcpyHostToDevice, ctx->copy_stream));
        ctx->h2d_bytes += (uint64_t)m * 8;
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
        CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0));
        if ((rc = launch((const int32_t*)dst, m))) return rc;
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
    }
    return CHP_OK;
}

// Host side of the packed pipeline: (x, y) -> slot | (y - 1) << 16 for a
// slice, returning nonzero if any point is invalid (slot >= wcheck or y
// outside [1, q]).  SSE2, 4 points per step, non-temporal stores: the pinned
// staging is only read by the DMA engine, so skipping the read-for-ownership
// saves a third of the host memory traffic.
uint32_t pack16_sse2(const int32_t* __restrict__ src, uint32_t* __restrict__ dst, uint64_t m, uint32_t base,
                     uint32_t ybase, uint32_t wcheck, uint32_t qmax) {
    uint32_t bad = 0;
    uint64_t i = 0;
    auto one = [&](uint64_t k) {
        const uint32_t s = (uint32_t)src[2 * k] - base;
        const uint32_t ym1 = (uint32_t)src[2 * k + 1] - ybase;
        bad |= (uint32_t)(s >= wcheck) | (uint32_t)(ym1 >= qmax);
        dst[k] = s | (ym1 << 16);
    };
    for (; i < m && (reinterpret_cast<uintptr_t>(dst + i) & 15); ++i) one(i);
    const __m128i vbase = _mm_set1_epi32((int)base), vone = _mm_set1_epi32((int)ybase);
    const __m128i sign = _mm_set1_epi32((int)0x80000000u);
    const __m128i wlim = _mm_set1_epi32((int)(wcheck ^ 0x80000000u)), qlim = _mm_set1_epi32((int)(qmax ^ 0x80000000u));
    __m128i okv = _mm_set1_epi32(-1);
    for (; i + 4 <= m; i += 4) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 2 * i));      // x0 y0 x1 y1
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 2 * i + 4));  // x2 y2 x3 y3
        const __m128i a2 = _mm_shuffle_epi32(a, _MM_SHUFFLE(3, 1, 2, 0));                     // x0 x1 y0 y1
        const __m128i b2 = _mm_shuffle_epi32(b, _MM_SHUFFLE(3, 1, 2, 0));                     // x2 x3 y2 y3
        const __m128i s = _mm_sub_epi32(_mm_unpacklo_epi64(a2, b2), vbase);
        const __m128i ym1 = _mm_sub_epi32(_mm_unpackhi_epi64(a2, b2), vone);
        // unsigned v < lim  <=>  signed (v ^ 2^31) < (lim ^ 2^31)
        okv = _mm_and_si128(okv, _mm_cmplt_epi32(_mm_xor_si128(s, sign), wlim));
        okv = _mm_and_si128(okv, _mm_cmplt_epi32(_mm_xor_si128(ym1, sign), qlim));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), _mm_or_si128(s, _mm_slli_epi32(ym1, 16)));
    }
    for (; i < m; ++i) one(i);
    _mm_sfence();  // the stores are weakly ordered; the DMA is enqueued after this returns
    return bad | (uint32_t)(_mm_movemask_epi8(okv) != 0xFFFF);
}

// AVX2 form (8 points per step): tools/micro_pack.cpp measured 11.7 vs 9.5
// Gpts/s for SSE2 on the 16-core GPU host.  Unsigned range checks as
// max_epu32(v, lim) == v  <=>  v >= lim.
__attribute__((target("avx2"))) uint32_t pack16_avx2(const int32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                     uint64_t m, uint32_t base, uint32_t ybase, uint32_t wcheck,
                                                     uint32_t qmax) {
    uint64_t i = 0;
    uint32_t bad = 0;
    for (; i < m && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) {
        const uint32_t s = (uint32_t)src[2 * i] - base;
        const uint32_t ym1 = (uint32_t)src[2 * i + 1] - ybase;
        bad |= (uint32_t)(s >= wcheck) | (uint32_t)(ym1 >= qmax);
        dst[i] = s | (ym1 << 16);
    }
    const __m256i vbase = _mm256_set1_epi32((int)base), vone = _mm256_set1_epi32((int)ybase);
    const __m256i wl = _mm256_set1_epi32((int)wcheck), ql = _mm256_set1_epi32((int)qmax);
    const __m256i perm = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
    __m256i badv = _mm256_setzero_si256();
    for (; i + 8 <= m; i += 8) {
        // x0 y0 .. x3 y3 | x4 y4 .. x7 y7 -> x0..x3 y0..y3 | x4..x7 y4..y7
        const __m256i a = _mm256_permutevar8x32_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 2 * i)), perm);
        const __m256i b =
            _mm256_permutevar8x32_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 2 * i + 8)), perm);
        const __m256i s = _mm256_sub_epi32(_mm256_permute2x128_si256(a, b, 0x20), vbase);
        const __m256i ym1 = _mm256_sub_epi32(_mm256_permute2x128_si256(a, b, 0x31), vone);
        badv = _mm256_or_si256(badv, _mm256_cmpeq_epi32(_mm256_max_epu32(s, wl), s));
        badv = _mm256_or_si256(badv, _mm256_cmpeq_epi32(_mm256_max_epu32(ym1, ql), ym1));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), _mm256_or_si256(s, _mm256_slli_epi32(ym1, 16)));
    }
    for (; i < m; ++i) {
        const uint32_t s = (uint32_t)src[2 * i] - base;
        const uint32_t ym1 = (uint32_t)src[2 * i + 1] - ybase;
        bad |= (uint32_t)(s >= wcheck) | (uint32_t)(ym1 >= qmax);
        dst[i] = s | (ym1 << 16);
    }
    _mm_sfence();
    return bad | (uint32_t)!_mm256_testz_si256(badv, badv);
}

uint32_t pack16(const int32_t* src, uint32_t* dst, uint64_t m, uint32_t base, uint32_t ybase, uint32_t wcheck,
                uint32_t qmax) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    return avx2 ? pack16_avx2(src, dst, m, base, ybase, wcheck, qmax)
                : pack16_sse2(src, dst, m, base, ybase, wcheck, qmax);
}

// pack16 for any host array: the SIMD forms for int32 input, a scalar loop
// with 64-bit range checks for int64 input (anything outside the window,
// including a value beyond int32, is flagged).
uint32_t pack_any(const HostPts& in, uint64_t off, uint64_t m, uint32_t* __restrict__ dst, uint32_t base,
                  uint32_t ybase, uint32_t wcheck, uint32_t qmax) {
    if (in.p32) return pack16(in.p32 + 2 * off, dst, m, base, ybase, wcheck, qmax);
    const int64_t b64 = (int32_t)base, y64 = (int32_t)ybase;
    uint32_t bad = 0;
    for (uint64_t k = 0; k < m; ++k) {
        const int64_t s = in.x(off + k) - b64, t = in.y(off + k) - y64;
        bad |= (uint32_t)((uint64_t)s >= wcheck) | (uint32_t)((uint64_t)t >= qmax);
        dst[k] = (uint32_t)s | ((uint32_t)t << 16);
    }
    return bad;
}

// 8-bit packing (width and y range up to 2^8 each, e.g. C5's 256 x 256):
// v = slot | (y - ybase) << 8 as uint16, eight points per 16-byte word, 2
// bytes per point instead of 8 (k_unpack8 in misc.cu).  16 points per AVX2
// step: the (x, y) lanes are split, range-checked and combined as in
// pack16_avx2, then two 8 x 32-bit vectors narrow to one 16 x 16-bit store
// (packus saturates only invalid points, which are flagged anyway).
__attribute__((target("avx2"))) uint32_t pack8_avx2(const int32_t* __restrict__ src, uint16_t* __restrict__ dst,
                                                    uint64_t m, uint32_t base, uint32_t ybase, uint32_t wcheck,
                                                    uint32_t qmax) {
    uint64_t i = 0;
    uint32_t bad = 0;
    auto one = [&](uint64_t k) {
        const uint32_t s = (uint32_t)src[2 * k] - base;
        const uint32_t t = (uint32_t)src[2 * k + 1] - ybase;
        bad |= (uint32_t)(s >= wcheck) | (uint32_t)(t >= qmax);
        dst[k] = (uint16_t)((s & 0xFFu) | ((t & 0xFFu) << 8));
    };
    for (; i < m && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) one(i);
    const __m256i vbase = _mm256_set1_epi32((int)base), vone = _mm256_set1_epi32((int)ybase);
    const __m256i wl = _mm256_set1_epi32((int)wcheck), ql = _mm256_set1_epi32((int)qmax);
    const __m256i perm = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
    __m256i badv = _mm256_setzero_si256();
    for (; i + 16 <= m; i += 16) {
        const __m256i* p = reinterpret_cast<const __m256i*>(src + 2 * i);
        const __m256i a = _mm256_permutevar8x32_epi32(_mm256_loadu_si256(p), perm);
        const __m256i b = _mm256_permutevar8x32_epi32(_mm256_loadu_si256(p + 1), perm);
        const __m256i c = _mm256_permutevar8x32_epi32(_mm256_loadu_si256(p + 2), perm);
        const __m256i d = _mm256_permutevar8x32_epi32(_mm256_loadu_si256(p + 3), perm);
        const __m256i s0 = _mm256_sub_epi32(_mm256_permute2x128_si256(a, b, 0x20), vbase);
        const __m256i t0 = _mm256_sub_epi32(_mm256_permute2x128_si256(a, b, 0x31), vone);
        const __m256i s1 = _mm256_sub_epi32(_mm256_permute2x128_si256(c, d, 0x20), vbase);
        const __m256i t1 = _mm256_sub_epi32(_mm256_permute2x128_si256(c, d, 0x31), vone);
        badv = _mm256_or_si256(badv, _mm256_cmpeq_epi32(_mm256_max_epu32(s0, wl), s0));
        badv = _mm256_or_si256(badv, _mm256_cmpeq_epi32(_mm256_max_epu32(t0, ql), t0));
        badv = _mm256_or_si256(badv, _mm256_cmpeq_epi32(_mm256_max_epu32(s1, wl), s1));
        badv = _mm256_or_si256(badv, _mm256_cmpeq_epi32(_mm256_max_epu32(t1, ql), t1));
        const __m256i w0 = _mm256_or_si256(s0, _mm256_slli_epi32(t0, 8));
        const __m256i w1 = _mm256_or_si256(s1, _mm256_slli_epi32(t1, 8));
        // packus: [w0 0-3 | w1 0-3 | w0 4-7 | w1 4-7] -> qwords 0, 2, 1, 3
        const __m256i pk = _mm256_permute4x64_epi64(_mm256_packus_epi32(w0, w1), 0xD8);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), pk);
    }
    for (; i < m; ++i) one(i);
    _mm_sfence();
    return bad | (uint32_t)!_mm256_testz_si256(badv, badv);
}

uint32_t pack8_any(const HostPts& in, uint64_t off, uint64_t m, uint16_t* __restrict__ dst, uint32_t base,
                   uint32_t ybase, uint32_t wcheck, uint32_t qmax) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (in.p32 && avx2) return pack8_avx2(in.p32 + 2 * off, dst, m, base, ybase, wcheck, qmax);
    const int64_t b64 = (int32_t)base, y64 = (int32_t)ybase;
    uint32_t bad = 0;
    for (uint64_t k = 0; k < m; ++k) {
        const int64_t s = in.x(off + k) - b64, t = in.y(off + k) - y64;
        bad |= (uint32_t)((uint64_t)s >= wcheck) | (uint32_t)((uint64_t)t >= qmax);
        dst[k] = (uint16_t)(((uint32_t)s & 0xFFu) | (((uint32_t)t & 0xFFu) << 8));
    }
    return bad;
}

// 42-bit packing (width and y range up to 2^21 each, e.g. C4's 2^20 x 2^20):
// v = slot | (y - ybase) << 21, three points per 16-byte word (lo64 = v0 |
// v1 << 42, hi64 = v1 >> 22 | v2 << 20; k_unpack42 in misc.cu), 5.33 bytes
// per point instead of 8.  m need not be a multiple of 3 (the last word is
// zero-padded); dst holds (m + 2) / 3 words.
uint32_t pack42_any(const HostPts& in, uint64_t off, uint64_t m, uint64_t* __restrict__ dst, uint32_t base,
                    uint32_t ybase, uint32_t wcheck, uint32_t qmax) {
    uint32_t bad = 0;
    auto val = [&](uint64_t k) -> uint64_t {
        uint64_t s, t;
        if (in.p32) {
            s = (uint32_t)in.p32[2 * (off + k)] - base;
            t = (uint32_t)in.p32[2 * (off + k) + 1] - ybase;
        } else {
            s = (uint64_t)(in.x(off + k) - (int64_t)(int32_t)base);
            t = (uint64_t)(in.y(off + k) - (int64_t)(int32_t)ybase);
        }
        bad |= (uint32_t)(s >= wcheck) | (uint32_t)(t >= qmax);
        return (s & 0x1FFFFF) | ((t & 0x1FFFFF) << 21);
    };
    const uint64_t full = m / 3;
    for (uint64_t w = 0; w < full; ++w) {
        const uint64_t v0 = val(3 * w), v1 = val(3 * w + 1), v2 = val(3 * w + 2);
        const __m128i q = _mm_set_epi64x((long long)((v1 >> 22) | (v2 << 20)), (long long)(v0 | (v1 << 42)));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 2 * w), q);
    }
    if (m % 3) {
        uint64_t v[3] = {0, 0, 0};
        for (uint64_t k = 3 * full; k < m; ++k) v[k - 3 * full] = val(k);
        dst[2 * full] = v[0] | (v[1] << 42);
        dst[2 * full + 1] = (v[1] >> 22) | (v[2] << 20);
    }
    _mm_sfence();
    return bad;
}

// Packed form of stream_chunks for width <= 2^16 and 1 <= y <= q <= 2^16:
// host workers pack chunk k into pinned 4-byte/point staging while the DMA
// of chunk k-1 is in flight, so PCIe carries half the bytes; on the device
// k_unpack16 restores int32 pairs and launch() consumes them.  *bad is set
// when any point is invalid (the caller fails the call).
//
// When the host packs slower than PCIe drains (16-core host: ~9-12 Gpts/s,
// bound by host memory bandwidth once the DMA reads compete, vs ~13.7 Gpts/s
// of packed words) and the input is pinned, the copy
// engine would idle during each pack; it is kept busy with int32 chunks
// DMA'd straight from the END of the input (K1 validates those itself), so
// the packed front and the raw back meet where both resources finish.
//
// mode: kPack16 (4 bytes per point), kPack42 (three points per 16-byte word,
// ranges up to 2^21 x 2^21), kPack8 (2 bytes per point, ranges up to
// 2^8 x 2^8).  Each is used both for known ranges (reduce with q given) and
// speculatively against a window (reduce with q unset: kPack16;
// precondition: the window its input's prefix fits, any mode): a chunk that
// fails the window check then travels as int32 pairs (send_raw).
enum PackMode { kPack16 = 0, kPack42 = 1, kPack8 = 2 };
template <typename Launch>
int stream_chunks_packed(chp_ctx* ctx, const HostPts& in, uint64_t n, int64_t x_off, int32_t ybase,
                         uint32_t wcheck, uint32_t qmax, bool speculative, bool* bad, Launch&& launch,
                         int32_t* d_dest = nullptr, int mode = kPack16) {
    *bad = false;
    if (n == 0) return CHP_OK;
    const bool wide = mode == kPack42;
    // packed bytes of m points; part boundaries within a chunk keep whole words
    auto pbytes = [&](uint64_t m) -> uint64_t {
        return wide ? (m + 2) / 3 * 16 : mode == kPack8 ? (m + 7) / 8 * 16 : m * 4;
    };
    const uint64_t align = wide ? 24 : 16;
    double& rate = wide ? ctx->pack_rate42 : mode == kPack8 ? ctx->pack_rate8 : ctx->pack_rate;
    // 8 Mi points per chunk (e2e C2, hybrid: 2 Mi 8.7-9.1, 4 Mi 9.4-9.7, 8 Mi
    // 9.9, 16 Mi 10.0 Gpts/s; smaller chunks pay the per-chunk dispatch).
    constexpr uint64_t kPackChunk = 8ull << 20;
    constexpr double kPcieBps = 50e9;  // H2D bytes / s (PCIe 5 x16, measured ~55e9)
    // (42-bit: whole 3-point words per chunk, so only the input's last word pads)
    const uint64_t chunk = std::min<uint64_t>(wide ? kPackChunk / 24 * 24 : kPackChunk, n);
    const bool pinned = in.pinned32();
    const bool hybrid = pinned;
    int rc;
    for (int b = 0; b < 2; ++b) {
        if ((rc = chp_ensure(ctx, ctx->stage_dev[b], (size_t)pbytes(chunk)))) return rc;
        if ((rc = chp_ensure(ctx, ctx->unpack_dev[b], (size_t)chunk * 8))) return rc;
        if ((hybrid || speculative) && (rc = chp_ensure(ctx, ctx->raw_dev[b], (size_t)chunk * 8))) return rc;
        if ((hybrid || speculative) && !ctx->ev_rcopied[b]) {
            CHP_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_rcopied[b], cudaEventDisableTiming));
            CHP_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_rconsumed[b], cudaEventDisableTiming));
        }
    }
    if (ctx->pack_bytes < (size_t)pbytes(chunk)) {
        for (int b = 0; b < 2; ++b) {
            if (ctx->pack_host[b]) cudaFreeHost(ctx->pack_host[b]);
            ctx->pack_host[b] = nullptr;
        }
        for (int b = 0; b < 2; ++b) CHP_CUDA(ctx, cudaMallocHost(&ctx->pack_host[b], (size_t)pbytes(chunk)));
        ctx->pack_bytes = (size_t)pbytes(chunk);
    }
    HostPool* pool = pool_of(ctx);
    const uint32_t base = (uint32_t)(int32_t)(x_off + 1);
    if (speculative && !pinned && ctx->stage_bytes < (size_t)chunk * 8) {
        for (int b = 0; b < 2; ++b) {
            if (ctx->stage_host[b]) cudaFreeHost(ctx->stage_host[b]);
            ctx->stage_host[b] = nullptr;
        }
        for (int b = 0; b < 2; ++b) CHP_CUDA(ctx, cudaMallocHost(&ctx->stage_host[b], (size_t)chunk * 8));
        ctx->stage_bytes = (size_t)chunk * 8;
    }
    for (int b = 0; b < 2; ++b) {
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
        if (hybrid || speculative) {
            CHP_CUDA(ctx, cudaEventRecord(ctx->ev_rconsumed[b], ctx->stream));
            CHP_CUDA(ctx, cudaEventRecord(ctx->ev_rcopied[b], ctx->copy_stream));
        }
    }
    uint32_t any_bad = 0, narrow_bad = 0;
    std::vector<uint32_t> part_bad((size_t)pool->parts());
    uint64_t front = 0, back = n;  // packed: [0, front); raw: [back, n)
    uint64_t k = 0, kr = 0;
    // Raw int32 chunks from the back covering `secs` of copy-engine time.
    auto raw_fill = [&](double secs) -> int {
        uint64_t want = (uint64_t)(secs * kPcieBps / 8);
        while (want > 0 && back > front) {
            const int rb = (int)(kr++ & 1);
            const uint64_t m = std::min<uint64_t>({want, chunk, back - front});
            const uint64_t off = back - m;
            CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_rconsumed[rb], 0));
            int32_t* rdst = d_dest ? d_dest + 2 * off : (int32_t*)ctx->raw_dev[rb].p;
            CHP_CUDA(ctx, cudaMemcpyAsync(rdst, in.p32 + 2 * off, (size_t)m * 8, cudaMemcpyHostToDevice,
                                          ctx->copy_stream));
            ctx->h2d_bytes += (uint64_t)m * 8;
            CHP_CUDA(ctx, cudaEventRecord(ctx->ev_rcopied[rb], ctx->copy_stream));
            CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_rcopied[rb], 0));
            int r = launch((const int32_t*)rdst, m);
            if (r) return r;
            CHP_CUDA(ctx, cudaEventRecord(ctx->ev_rconsumed[rb], ctx->stream));
            back = off;
            want -= m;
        }
        return CHP_OK;
    };
    // One int32 chunk [off, off+m) to the device and through K1 (which
    // validates it): a speculatively packed chunk that did not fit 16 bits.
    auto send_raw = [&](uint64_t off, uint64_t m) -> int {
        const int rb = (int)(kr++ & 1);
        const int32_t* src = in.p32 ? in.p32 + 2 * off : nullptr;
        if (!pinned) {
            CHP_CUDA(ctx, cudaEventSynchronize(ctx->ev_rcopied[rb]));
            narrow_bad |= stage_copy(ctx, in, off, m, static_cast<int32_t*>(ctx->stage_host[rb]));
            src = static_cast<const int32_t*>(ctx->stage_host[rb]);
        }
        CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_rconsumed[rb], 0));
        int32_t* rdst = d_dest ? d_dest + 2 * off : (int32_t*)ctx->raw_dev[rb].p;
        CHP_CUDA(ctx, cudaMemcpyAsync(rdst, src, (size_t)m * 8, cudaMemcpyHostToDevice, ctx->copy_stream));
        ctx->h2d_bytes += (uint64_t)m * 8;
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_rcopied[rb], ctx->copy_stream));
        CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_rcopied[rb], 0));
        int r = launch((const int32_t*)rdst, m);
        if (r) return r;
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_rconsumed[rb], ctx->stream));
        return CHP_OK;
    };
    double dma_ahead = 0;  // copy-engine seconds already queued when a pack starts
    while (front < back) {
        const uint64_t m = std::min<uint64_t>(chunk, back - front);
        if (hybrid) {
            // Keep the copy engine busy for the duration of this pack.
            const double t_pack = (double)m / rate;
            if (t_pack > dma_ahead && (rc = raw_fill(t_pack - dma_ahead))) return rc;
            if (front >= back) break;
        }
        const uint64_t mm = std::min<uint64_t>(m, back - front);
        const int b = (int)(k++ & 1);
        // The DMA out of this staging buffer (two packed chunks ago) must be done.
        CHP_CUDA(ctx, cudaEventSynchronize(ctx->ev_copied[b]));
        uint32_t* dst = static_cast<uint32_t*>(ctx->pack_host[b]);
        uint64_t* dst64 = static_cast<uint64_t*>(ctx->pack_host[b]);
        uint16_t* dst16 = static_cast<uint16_t*>(ctx->pack_host[b]);
        const int parts = pool->parts_for(mm);
        const auto t0 = std::chrono::steady_clock::now();
        std::fill(part_bad.begin(), part_bad.end(), 0u);
        pool->run(
            [&](int i) {
                const uint64_t lo = mm * (uint64_t)i / parts / align * align;
                const uint64_t hi = i + 1 == parts ? mm : mm * (uint64_t)(i + 1) / parts / align * align;
                part_bad[(size_t)i] =
                    wide ? pack42_any(in, front + lo, hi - lo, dst64 + 2 * (lo / 3), base, (uint32_t)ybase, wcheck, qmax)
                    : mode == kPack8
                        ? pack8_any(in, front + lo, hi - lo, dst16 + lo, base, (uint32_t)ybase, wcheck, qmax)
                        : pack_any(in, front + lo, hi - lo, dst + lo, base, (uint32_t)ybase, wcheck, qmax);
            },
            parts);
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (mm >= (1u << 20) && dt > 0) rate = 0.5 * rate + 0.5 * (double)mm / dt;
        uint32_t chunk_bad = 0;
        for (uint32_t v : part_bad) chunk_bad |= v;
        if (chunk_bad && speculative) {  // not 16-bit: the chunk goes as int32 pairs
            if ((rc = send_raw(front, mm))) return rc;
            front += mm;
            dma_ahead = (double)mm * 8 / kPcieBps;
            continue;
        }
        any_bad |= chunk_bad;
        CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_consumed[b], 0));
        CHP_CUDA(ctx, cudaMemcpyAsync(ctx->stage_dev[b].p, dst, (size_t)pbytes(mm), cudaMemcpyHostToDevice,
                                      ctx->copy_stream));
        ctx->h2d_bytes += pbytes(mm);
        dma_ahead = (double)pbytes(mm) / kPcieBps;
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
        CHP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0));
        int32_t* udst = d_dest ? d_dest + 2 * front : (int32_t*)ctx->unpack_dev[b].p;
        if ((rc = wide ? chp_unpack42(ctx, ctx->stage_dev[b].p, mm, (int32_t)base, ybase, udst)
                  : mode == kPack8 ? chp_unpack8(ctx, ctx->stage_dev[b].p, mm, (int32_t)base, ybase, udst)
                                   : chp_unpack16(ctx, (const uint32_t*)ctx->stage_dev[b].p, mm, (int32_t)base,
                                                  ybase, udst)))
            return rc;
        CHP_CUDA(ctx, cudaEventRecord(ctx->ev_consumed[b], ctx->stream));
        if ((rc = launch(d_dest ? (const int32_t*)(d_dest + 2 * front) : (const int32_t*)ctx->unpack_dev[b].p, mm)))
            return rc;
        front += mm;
    }
    *bad = (any_bad | narrow_bad) != 0;
    return CHP_OK;
}

// A 2^16 x 2^16 packing window from the box of the first min(n, 64 Ki)
// points, centred in the slack; false when that prefix is already wider or
// taller than 2^16.
bool pack_window(chp_ctx* ctx, const HostPts& in, uint64_t n, int64_t* wx, int64_t* wy, int64_t W = 65536) {
    (void)ctx;
    const uint64_t m = std::min<uint64_t>(n, 1ull << 16);  // a 64 Ki-point prefix, on the caller's thread
    int64_t b[4] = {INT64_MAX, INT64_MIN, INT64_MAX, INT64_MIN};
    for (uint64_t k = 0; k < m; ++k) {
        const int64_t x = in.x(k), y = in.y(k);
        b[0] = std::min(b[0], x);
        b[1] = std::max(b[1], x);
        b[2] = std::min(b[2], y);
        b[3] = std::max(b[3], y);
    }
    auto place = [W](int64_t lo, int64_t hi, int64_t* base) {
        const int64_t ext = hi - lo + 1;
        if (ext > W || lo < INT32_MIN || hi > INT32_MAX) return false;
        int64_t s = lo - (W - ext) / 2;
        s = std::max<int64_t>(s, INT32_MIN);
        s = std::min<int64_t>(s, (int64_t)INT32_MAX - (W - 1));
        *base = s;
        return true;
    };
    return place(b[0], b[1], wx) && place(b[2], b[3], wy);
}

// Streams h_xy[0..n) into ctx->dl (accumulating; it must be initialised),
// valid y in [ybase, ybase + ycount) (ycount < 0: no upper bound).  Inputs
// whose slots and y offsets fit 16 bits travel packed (half the PCIe bytes)
// unless CHP_PIPELINE_NO_PACK is set in flags or the environment.
int stream_reduce(chp_ctx* ctx, const HostPts& in, uint64_t n, int64_t width, int64_t ybase, int64_t ycount,
                  int64_t x_off, uint32_t flags, int32_t* d_L = nullptr) {
    if (!d_L) d_L = (int32_t*)ctx->dl.p;
    auto launch = [&](const int32_t* d, uint64_t m) {
        return chp_reduce_yr(ctx, d, m, width, ybase, ycount, x_off, d_L, flags | CHP_REDUCE_ACCUMULATE);
    };
    // ycount < 0 (no upper bound, the reference's default q = nullopt):
    // pack speculatively against a 2^16 window; chunks with a larger y go
    // as int32 pairs and K1 validates them.
    const bool speculative = ycount < 0;
    const bool packable = width <= 65536 && (speculative || ycount <= 65536) && ycount != 0 &&
                          !(flags & CHP_REDUCE_NO_VALIDATE) &&
                          !(flags & CHP_PIPELINE_NO_PACK) && !std::getenv("CHP_PIPELINE_NO_PACK") &&
                          x_off + 1 >= (int64_t)INT32_MIN && x_off <= (int64_t)INT32_MAX &&
                          ybase >= (int64_t)INT32_MIN && ybase <= (int64_t)INT32_MAX;
    // Known ranges up to 2^21 x 2^21 (e.g. C4: 2^20 x 2^20): the 42-bit form.
    const bool packable42 = !packable && !speculative && width <= (1 << 21) && ycount >= 1 && ycount <= (1 << 21) &&
                            !(flags & CHP_REDUCE_NO_VALIDATE) && !(flags & CHP_PIPELINE_NO_PACK) &&
                            !std::getenv("CHP_PIPELINE_NO_PACK") && x_off + 1 >= (int64_t)INT32_MIN &&
                            x_off <= (int64_t)INT32_MAX && ybase >= (int64_t)INT32_MIN && ybase <= (int64_t)INT32_MAX;
    // Known ranges up to 2^8 x 2^8 (e.g. C5: 256 x 256): 2 bytes per point.
    const bool packable8 = packable && !speculative && width <= 256 && ycount <= 256;
    bool bad = false;
    int rc;
    if (!packable && !packable42) {
        uint32_t nb = 0;  // int64 input: a coordinate beyond int32
        if ((rc = stream_chunks(ctx, in, n, launch, nullptr, &nb))) return rc;
        bad = nb != 0;
    } else {
        const uint32_t wcheck = (uint32_t)std::min<int64_t>(width, (int64_t)INT32_MAX - x_off);
        const uint32_t qmax =
            (uint32_t)std::min<int64_t>(speculative ? 65536 : ycount, (int64_t)INT32_MAX - ybase + 1);
        if ((rc = stream_chunks_packed(ctx, in, n, x_off, (int32_t)ybase, wcheck, qmax, speculative, &bad, launch,
                                       nullptr, packable8 ? kPack8 : packable42 ? kPack42 : kPack16)))
            return rc;
    }
    if (bad) {  // same outcome as the unpacked path: the error word of DL
        int32_t minus1 = -1;
        CHP_CUDA(ctx, cudaMemcpyAsync(d_L + 2 * width, &minus1, 4, cudaMemcpyHostToDevice,
                                      ctx->stream));
        CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return CHP_OK;
}

// Compaction (+ hull) of d_L (default ctx->dl) into the context's device
// buffers; cnt receives the K3/K4 counts {s, v, err, s-v, h}.
int finish_device(chp_ctx* ctx, int64_t width, int64_t major_off, int64_t minor_off, bool want_chain,
                  bool want_lpairs, bool want_occ, bool want_hull, int64_t cnt[8], const int32_t* d_L = nullptr) {
    if (!d_L) d_L = (const int32_t*)ctx->dl.p;
    int rc;
    const size_t W = (size_t)width;
    if ((rc = chp_ensure(ctx, ctx->counts, 16 * sizeof(int64_t)))) return rc;
    if ((rc = chp_ensure(ctx, ctx->chain, 2 * W * 8))) return rc;
    if ((rc = chp_ensure(ctx, ctx->occ, ((W + 63) / 64) * 8))) return rc;
    if ((rc = chp_ensure(ctx, ctx->lpairs, W * 8))) return rc;
    if (want_hull) {
        if ((rc = chp_ensure(ctx, ctx->lower, W * 8))) return rc;
        if ((rc = chp_ensure(ctx, ctx->upper, W * 8))) return rc;
        if ((rc = chp_ensure(ctx, ctx->hull, (2 * W + 4) * 8))) return rc;
    }
    int64_t* d_counts = (int64_t*)ctx->counts.p;
    if ((rc = chp_compact(ctx, d_L, width, major_off, minor_off, 0,
                          want_chain ? (int32_t*)ctx->chain.p : nullptr, want_occ ? (uint64_t*)ctx->occ.p : nullptr,
                          want_lpairs ? (int32_t*)ctx->lpairs.p : nullptr,
                          want_hull ? (int32_t*)ctx->lower.p : nullptr,
                          want_hull ? (int32_t*)ctx->upper.p : nullptr, nullptr, d_counts)))
        return rc;
    if (want_hull) {
        if ((rc = chp_hull(ctx, (const int32_t*)ctx->lower.p, (const int32_t*)ctx->upper.p, d_counts, width, 0,
                           (int32_t*)ctx->hull.p, d_counts + 4)))
            return rc;
    }
    CHP_CUDA(ctx, cudaMemcpyAsync(cnt, d_counts, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (!want_hull) cnt[4] = 0;
    return CHP_OK;
}

// The context's device results to host buffers (any may be NULL).
int copy_out(chp_ctx* ctx, int64_t width, int64_t s, int64_t h, int32_t* h_Lpairs, uint64_t* h_occ,
             int32_t* h_chain, int32_t* h_hull) {
    const size_t W = (size_t)width;
    if (h_Lpairs)
        CHP_CUDA(ctx, cudaMemcpyAsync(h_Lpairs, ctx->lpairs.p, W * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_occ)
        CHP_CUDA(ctx, cudaMemcpyAsync(h_occ, ctx->occ.p, ((W + 63) / 64) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_chain && s > 0)
        CHP_CUDA(ctx, cudaMemcpyAsync(h_chain, ctx->chain.p, (size_t)s * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_hull && h > 0)
        CHP_CUDA(ctx, cudaMemcpyAsync(h_hull, ctx->hull.p, (size_t)h * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return CHP_OK;
}

// Compaction (+ hull) of d_L (default ctx->dl), then the requested outputs
// to the host.
int finish_host(chp_ctx* ctx, int64_t width, int64_t major_off, int64_t minor_off, int32_t* h_Lpairs,
                uint64_t* h_occ, int32_t* h_chain, int64_t* h_s, int32_t* h_hull, int64_t* h_h,
                bool chain_required, const int32_t* d_L = nullptr) {
    int64_t cnt[8];
    const bool want_hull = h_hull || h_h;
    int rc = finish_device(ctx, width, major_off, minor_off, h_chain || h_s, h_Lpairs != nullptr, h_occ != nullptr,
                           want_hull, cnt, d_L);
    if (rc) return rc;
    if (cnt[2] != 0) return chp_einval(ctx, "reduce: coordinate out of range");
    const int64_t s = cnt[0];
    if (h_s) *h_s = s;
    if (s == 0 && chain_required) return chp_einval(ctx, "build_polyline: no valid points");
    if (want_hull && h_h) *h_h = cnt[4];
    return copy_out(ctx, width, s, cnt[4], h_Lpairs, h_occ, h_chain, h_hull);
}

}  // namespace

extern "C" {

int chp_ctx_create(int device, chp_ctx** out) {
    if (!out) return CHP_EINVAL;
    *out = nullptr;
    chp_ctx* ctx = new chp_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_switch, cudaEventDisableTiming);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_consumed[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess)
        e = cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->l2_bytes, cudaDevAttrL2CacheSize, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->coop, cudaDevAttrCooperativeLaunch, device);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return CHP_EDEVICE;
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return CHP_OK;
}

void chp_ctx_destroy(chp_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->copy_stream);
    DevBuf* bufs[] = {&ctx->tile_status, &ctx->hull_a, &ctx->hull_b, &ctx->hull_cnt_a, &ctx->hull_cnt_b,
                      &ctx->filter, &ctx->sample, &ctx->gridbar, &ctx->yrange, &ctx->dl, &ctx->counts, &ctx->chain, &ctx->lower, &ctx->upper,
                      &ctx->hull, &ctx->occ, &ctx->lpairs, &ctx->stage_dev[0], &ctx->stage_dev[1]};
    for (DevBuf* b : bufs) free_buf(*b);
    free_buf(ctx->unpack_dev[0]);
    free_buf(ctx->unpack_dev[1]);
    free_buf(ctx->points);
    free_buf(ctx->raw_dev[0]);
    free_buf(ctx->raw_dev[1]);
    for (int b = 0; b < 2; ++b) {
        if (ctx->ev_rcopied[b]) cudaEventDestroy(ctx->ev_rcopied[b]);
        if (ctx->ev_rconsumed[b]) cudaEventDestroy(ctx->ev_rconsumed[b]);
    }
    delete static_cast<HostPool*>(ctx->pool);
    for (int b = 0; b < 2; ++b) {
        if (ctx->pack_host[b]) cudaFreeHost(ctx->pack_host[b]);
        if (ctx->stage_host[b]) cudaFreeHost(ctx->stage_host[b]);
        if (ctx->ev_copied[b]) cudaEventDestroy(ctx->ev_copied[b]);
        if (ctx->ev_consumed[b]) cudaEventDestroy(ctx->ev_consumed[b]);
    }
    if (ctx->ev_switch) cudaEventDestroy(ctx->ev_switch);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

const char* chp_last_error(const chp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// The context's scratch (filter / sample tables, grid barrier, look-back
// status words, hull buffers, pipeline staging) is shared by every call, so
// a stream switch orders the new stream after everything the context has
// issued on the old one (and on its copy stream): a context's work never
// overlaps itself, whichever streams a caller hands it.
static int switch_stream(chp_ctx* ctx, cudaStream_t s) {
    if (s == ctx->stream) return CHP_OK;
    CHP_CUDA(ctx, cudaSetDevice(ctx->device));
    CHP_CUDA(ctx, cudaEventRecord(ctx->ev_switch, ctx->stream));
    CHP_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_switch, 0));
    CHP_CUDA(ctx, cudaEventRecord(ctx->ev_switch, ctx->copy_stream));
    CHP_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_switch, 0));
    ctx->stream = s;
    return CHP_OK;
}

int chp_ctx_set_stream(chp_ctx* ctx, void* stream) {
    if (!ctx) return CHP_EINVAL;
    return switch_stream(ctx, (cudaStream_t)stream);
}

int chp_ctx_use_own_stream(chp_ctx* ctx) {
    if (!ctx) return CHP_EINVAL;
    return switch_stream(ctx, ctx->own_stream);
}

void* chp_ctx_stream(const chp_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int chp_ctx_sync(chp_ctx* ctx) {
    if (!ctx) return CHP_EINVAL;
    CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return CHP_OK;
}

uint64_t chp_launch_count(const chp_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* chp_last_variant(const chp_ctx* ctx) { return ctx ? ctx->variant : "none"; }

uint64_t chp_last_h2d_bytes(const chp_ctx* ctx) { return ctx ? ctx->h2d_bytes : 0; }

static int pipeline_core(chp_ctx* ctx, const HostPts& in, uint64_t n, int64_t width, int64_t q,
                         int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s, int32_t* h_hull,
                         int64_t* h_h) {
    if (!ctx) return CHP_EINVAL;
    ctx->h2d_bytes = 0;
    ctx->last_valid = false;
    if (width < 1) return chp_einval(ctx, "reduce: width must be >= 1");
    if (width > (1ll << 29)) return chp_einval(ctx, "reduce: width exceeds the device limit 2^29");
    CHP_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc;
    if ((rc = chp_ensure(ctx, ctx->dl, chp_dl_len(width) * 4))) return rc;
    if ((rc = chp_dl_init(ctx, (int32_t*)ctx->dl.p, width))) return rc;
    if ((rc = stream_reduce(ctx, in, n, width, 1, q, 0, 0))) return rc;
    return finish_host(ctx, width, 0, 0, h_Lpairs, h_occ, h_chain, h_s, h_hull, h_h,
                       h_chain != nullptr || h_hull != nullptr);
}

int chp_pipeline_host(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int64_t width, int64_t q,
                      int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s, int32_t* h_hull,
                      int64_t* h_h) {
    HostPts in;
    in.p32 = h_xy;
    return pipeline_core(ctx, in, n, width, q, h_Lpairs, h_occ, h_chain, h_s, h_hull, h_h);
}

int chp_pipeline_host64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q,
                        int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s, int32_t* h_hull,
                        int64_t* h_h) {
    HostPts in;
    in.p64 = h_xy;
    return pipeline_core(ctx, in, n, width, q, h_Lpairs, h_occ, h_chain, h_s, h_hull, h_h);
}

static int reduce_host_core(chp_ctx* ctx, const HostPts& in, uint64_t n, int64_t width, int64_t q, int32_t* d_L,
                            bool init = true) {
    if (!ctx || !d_L) return CHP_EINVAL;
    ctx->h2d_bytes = 0;
    ctx->last_valid = false;
    if (width < 1) return chp_einval(ctx, "reduce: width must be >= 1");
    if (width > (1ll << 29)) return chp_einval(ctx, "reduce: width exceeds the device limit 2^29");
    CHP_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc;
    if (init && (rc = chp_dl_init(ctx, d_L, width))) return rc;
    if ((rc = stream_reduce(ctx, in, n, width, 1, q, 0, 0, d_L))) return rc;
    CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return CHP_OK;
}

int chp_reduce_host(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int64_t width, int64_t q, int32_t* d_L) {
    HostPts in;
    in.p32 = h_xy;
    return reduce_host_core(ctx, in, n, width, q, d_L);
}

int chp_reduce_host64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q, int32_t* d_L) {
    HostPts in;
    in.p64 = h_xy;
    return reduce_host_core(ctx, in, n, width, q, d_L);
}

// Shard groups (shard.cu), CHP_COMBINE_FUSED: fold host points into a DL
// that is already initialised (possibly another device's, over peer memory).
int chp_reduce_host_into(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int64_t width, int64_t q, int32_t* d_L) {
    HostPts in;
    in.p32 = h_xy;
    return reduce_host_core(ctx, in, n, width, q, d_L, false);
}

int chp_reduce_host64_into(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q, int32_t* d_L) {
    HostPts in;
    in.p64 = h_xy;
    return reduce_host_core(ctx, in, n, width, q, d_L, false);
}

int chp_finish_host(chp_ctx* ctx, const int32_t* d_L, int64_t width, int32_t* h_Lpairs, uint64_t* h_occ,
                    int32_t* h_chain, int64_t* h_s, int32_t* h_hull, int64_t* h_h) {
    if (!ctx || !d_L) return CHP_EINVAL;
    if (width < 1 || width > (1ll << 29)) return chp_einval(ctx, "compact: width out of range");
    CHP_CUDA(ctx, cudaSetDevice(ctx->device));
    return finish_host(ctx, width, 0, 0, h_Lpairs, h_occ, h_chain, h_s, h_hull, h_h,
                       h_chain != nullptr || h_hull != nullptr, d_L);
}

int chp_translate_host(chp_ctx* ctx, const int32_t* h_in, uint64_t n, int32_t dx, int32_t dy, int32_t* h_out) {
    if (!ctx) return CHP_EINVAL;
    ctx->h2d_bytes = 0;
    ctx->last_valid = false;
    if (n == 0) return CHP_OK;
    CHP_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBuf buf;
    int rc = chp_ensure(ctx, buf, (size_t)n * 8);
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(buf.p, h_in, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) {
        rc = chp_translate(ctx, (const int32_t*)buf.p, n, dx, dy, (int32_t*)buf.p);
        if (!rc) e = cudaMemcpyAsync(h_out, buf.p, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    }
    free_buf(buf);
    if (rc) return rc;
    if (e != cudaSuccess) return chp_cuda_fail(ctx, e, "translate_host");
    return CHP_OK;
}

int chp_polyline_host(chp_ctx* ctx, const int32_t* h_Lpairs, int64_t width, int64_t major_off, int64_t minor_off,
                      int swapped, int32_t* h_chain, int64_t* h_s) {
    if (!ctx) return CHP_EINVAL;
    ctx->h2d_bytes = 0;
    ctx->last_valid = false;
    if (width < 1 || width > (1ll << 29)) return chp_einval(ctx, "build_polyline: width must be in [1, 2^29]");
    CHP_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc;
    const size_t W = (size_t)width;
    if ((rc = chp_ensure(ctx, ctx->lpairs, W * 8))) return rc;
    if ((rc = chp_ensure(ctx, ctx->dl, chp_dl_len(width) * 4))) return rc;
    if ((rc = chp_ensure(ctx, ctx->chain, 2 * W * 8))) return rc;
    if ((rc = chp_ensure(ctx, ctx->counts, 16 * sizeof(int64_t)))) return rc;
    CHP_CUDA(ctx, cudaMemcpyAsync(ctx->lpairs.p, h_Lpairs, W * 8, cudaMemcpyHostToDevice, ctx->stream));
    if ((rc = chp_dl_from_pairs(ctx, (const int32_t*)ctx->lpairs.p, width, (int32_t*)ctx->dl.p))) return rc;
    int64_t* d_counts = (int64_t*)ctx->counts.p;
    if ((rc = chp_compact(ctx, (const int32_t*)ctx->dl.p, width, major_off, minor_off, swapped,
                          (int32_t*)ctx->chain.p, nullptr, nullptr, nullptr, nullptr, nullptr, d_counts)))
        return rc;
    int64_t cnt[4];
    CHP_CUDA(ctx, cudaMemcpyAsync(cnt, d_counts, sizeof cnt, cudaMemcpyDeviceToHost, ctx->stream));
    CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (h_s) *h_s = cnt[0];
    if (h_chain) {
        if (cnt[0] == 0) return chp_einval(ctx, "build_polyline: no valid points");
        CHP_CUDA(ctx, cudaMemcpy(h_chain, ctx->chain.p, (size_t)cnt[0] * 8, cudaMemcpyDeviceToHost));
    }
    return CHP_OK;
}

static int precondition_core(chp_ctx* ctx, const HostPts& in, uint64_t n, int64_t* h_bbox4, bool bounds_only,
                             const std::function<int(int64_t width, int64_t x_off)>& finish) {
    if (!ctx) return CHP_EINVAL;
    ctx->h2d_bytes = 0;
    ctx->last_valid = false;
    if (n == 0) return chp_einval(ctx, "precondition: empty input");
    CHP_CUDA(ctx, cudaSetDevice(ctx->device));
    // Step 1 (bounds).  The points stay resident for step 3 when they fit a
    // quarter of free memory (copied in chunks, the bounds of each chunk
    // computed as it lands; the buffer is kept in the context); otherwise
    // they are streamed twice.
    int rc;
    // (cudaMemGetInfo costs 0.1-0.4 ms: only asked when the held buffer is
    // too small.  CHP_PRECONDITION_STREAM forces the streamed form: tests.)
    bool resident = (size_t)n * 8 <= ctx->points.bytes;
    if (!resident) {
        size_t freeb = 0, totalb = 0;
        CHP_CUDA(ctx, cudaMemGetInfo(&freeb, &totalb));
        resident = (size_t)n * 8 <= (freeb + ctx->points.bytes) / 4;
    }
    if (std::getenv("CHP_PRECONDITION_STREAM")) resident = false;
    DevBuf& pts = ctx->points;
    if ((rc = chp_ensure(ctx, ctx->counts, 16 * sizeof(int64_t)))) return rc;
    int32_t* d_b4 = (int32_t*)((int64_t*)ctx->counts.p + 8);
    int32_t b4[4];
    if (resident) {
        if ((rc = chp_ensure(ctx, pts, (size_t)n * 8))) return rc;
        if ((rc = chp_bounds_init(ctx, d_b4))) return rc;
        auto fold = [&](const int32_t* d, uint64_t m) { return chp_bounds_accumulate(ctx, d, m, d_b4); };
        // The box is unknown until every point has been seen, so the 16-bit
        // packing is speculative: a window sized from the first 64 Ki points'
        // box (centred in the 2^16 slack) packs every chunk that fits, the
        // rest travel as int32 pairs; either way they land unpacked in the
        // resident buffer.
        // A prefix wider than 2^16 tries a 2^21 window and the 42-bit form.
        int64_t wx = 0, wy = 0;
        const bool pack = !std::getenv("CHP_PIPELINE_NO_PACK");
        // A prefix within 2^8 x 2^8 tries a 2^8 window and 2 bytes per point.
        const bool win8 = pack && pack_window(ctx, in, n, &wx, &wy, 256);
        const bool win = pack && !win8 && pack_window(ctx, in, n, &wx, &wy);
        const bool win42 = pack && !win8 && !win && pack_window(ctx, in, n, &wx, &wy, 1 << 21);
        bool narrow_bad = false;  // int64 input: a coordinate beyond int32
        if (win8 || win || win42) {
            const uint32_t W = win8 ? 256u : win ? 65536u : (1u << 21);
            if ((rc = stream_chunks_packed(ctx, in, n, wx - 1, (int32_t)wy, W, W, true, &narrow_bad, fold,
                                           (int32_t*)pts.p, win8 ? kPack8 : win42 ? kPack42 : kPack16)))
                return rc;
        } else {
            uint32_t nb = 0;
            if ((rc = stream_chunks(ctx, in, n, fold, (int32_t*)pts.p, &nb))) return rc;
            narrow_bad = nb != 0;
        }
        if (narrow_bad) return chp_einval(ctx, "precondition: coordinate does not fit int32");
        CHP_CUDA(ctx, cudaMemcpyAsync(b4, d_b4, 16, cudaMemcpyDeviceToHost, ctx->stream));
        CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    } else {
        if ((rc = chp_bounds_init(ctx, d_b4))) return rc;
        uint32_t nb = 0;
        if ((rc = stream_chunks(
                 ctx, in, n, [&](const int32_t* d, uint64_t m) { return chp_bounds_accumulate(ctx, d, m, d_b4); },
                 nullptr, &nb)))
            return rc;
        if (nb) return chp_einval(ctx, "precondition: coordinate does not fit int32");
        CHP_CUDA(ctx, cudaMemcpyAsync(b4, d_b4, 16, cudaMemcpyDeviceToHost, ctx->stream));
        CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    for (int i = 0; i < 4; ++i) h_bbox4[i] = b4[i];
    const int64_t width = (int64_t)b4[1] - b4[0] + 1;
    if (bounds_only) return CHP_OK;
    if (width > (1ll << 29)) return chp_einval(ctx, "precondition: x extent exceeds the device limit 2^29");
    const int64_t x_off = (int64_t)b4[0] - 1;  // major_offset, src/reducer.cpp:154
    if ((rc = chp_ensure(ctx, ctx->dl, chp_dl_len(width) * 4))) return rc;
    // Every point lies in the bounding box, so K1 runs with the box's y range
    // as the valid range: the filter variants (and, streamed, the 16-bit
    // packing) apply, and validation can never fire.
    // (A y range of 2^32 - 1 or more values does not fit the uint32 test:
    // then no validation and no y range, as the reference's bucket().)
    int64_t ybase = b4[2], ycount = (int64_t)b4[3] - b4[2] + 1;
    uint32_t rflags = 0;
    if (ycount >= (1ll << 32) - 1) {
        ybase = 1;
        ycount = -1;
        rflags = CHP_REDUCE_NO_VALIDATE;
    }
    if (resident) {
        rc = chp_reduce_yr(ctx, (const int32_t*)pts.p, n, width, ybase, ycount, x_off, (int32_t*)ctx->dl.p, rflags);
    } else {
        rc = chp_dl_init(ctx, (int32_t*)ctx->dl.p, width);
        if (!rc) rc = stream_reduce(ctx, in, n, width, ybase, ycount, x_off, rflags);
    }
    if (rc) return rc;
    return finish(width, x_off);
}


int chp_precondition_host(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int64_t* h_bbox4, int32_t* h_Lpairs,
                          int32_t* h_chain, int64_t* h_s, int32_t* h_hull, int64_t* h_h) {
    const bool bounds_only = !h_chain && !h_hull && !h_s && !h_Lpairs && !h_h;
    HostPts in;
    in.p32 = h_xy;
    return precondition_core(ctx, in, n, h_bbox4, bounds_only, [&](int64_t width, int64_t x_off) {
        return finish_host(ctx, width, x_off, 0, h_Lpairs, nullptr, h_chain, h_s, h_hull, h_h, true);
    });
}

static int precondition_run_core(chp_ctx* ctx, const HostPts& in, uint64_t n, int want_hull, int64_t* h_bbox4,
                                 int64_t* h_width, int64_t* h_s, int64_t* h_h) {
    if (ctx) ctx->last_valid = false;
    int64_t width = 0, s = 0, h = 0;
    const int rc = precondition_core(ctx, in, n, h_bbox4, false, [&](int64_t w, int64_t x_off) {
        int64_t cnt[8];
        int r = finish_device(ctx, w, x_off, 0, true, true, false, want_hull != 0, cnt);
        if (r) return r;
        if (cnt[2] != 0) return chp_einval(ctx, "reduce: coordinate out of range");
        if (cnt[0] == 0) return chp_einval(ctx, "build_polyline: no valid points");
        width = w;
        s = cnt[0];
        h = cnt[4];
        return CHP_OK;
    });
    if (rc) return rc;
    ctx->last_valid = true;
    ctx->last_width = width;
    ctx->last_s = s;
    ctx->last_h = want_hull ? h : -1;
    if (h_width) *h_width = width;
    if (h_s) *h_s = s;
    if (h_h) *h_h = want_hull ? h : 0;
    return CHP_OK;
}

int chp_precondition_run(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int want_hull, int64_t* h_bbox4,
                         int64_t* h_width, int64_t* h_s, int64_t* h_h) {
    HostPts in;
    in.p32 = h_xy;
    return precondition_run_core(ctx, in, n, want_hull, h_bbox4, h_width, h_s, h_h);
}

int chp_precondition_run64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int swap_axes, int want_hull,
                           int64_t* h_bbox4, int64_t* h_width, int64_t* h_s, int64_t* h_h) {
    HostPts in;
    in.p64 = h_xy;
    in.swap = swap_axes != 0;
    return precondition_run_core(ctx, in, n, want_hull, h_bbox4, h_width, h_s, h_h);
}

int chp_bounds_host64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t* h_bbox4) {
    HostPts in;
    in.p64 = h_xy;
    // K0 on the device over the narrowed points (bounds only)
    return precondition_core(ctx, in, n, h_bbox4, true, [](int64_t, int64_t) { return CHP_OK; });
}

int chp_last_outputs(chp_ctx* ctx, int32_t* h_Lpairs, int32_t* h_chain, int32_t* h_hull) {
    if (!ctx) return CHP_EINVAL;
    if (!ctx->last_valid) return chp_einval(ctx, "last_outputs: no chp_precondition_run result on this context");
    if (h_hull && ctx->last_h < 0) return chp_einval(ctx, "last_outputs: the run did not compute the hull");
    return copy_out(ctx, ctx->last_width, ctx->last_s, ctx->last_h < 0 ? 0 : ctx->last_h, h_Lpairs, nullptr, h_chain,
                    h_hull);
}

}  // extern "C"
