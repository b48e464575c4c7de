// reduce.cu -- K1: Algorithm 1 (per-x-column min/max of y) on sm_100a.
//
// Replaces reducer::reduce's validation pass and the bucket() fold
// (/root/reference/proj/src/reducer.cpp:172-182, :122-135).  The fold is a
// scatter-min over a p-slot table, so the kernel is HBM-bound on the 8-byte
// point stream when every per-point table access stays on chip:
//
//  smem32  : slot table privatised per CTA in shared memory, 8 B per slot
//            (lo, ~hi); read-compare-then-ATOMS, so a point that changes
//            nothing costs one LDS.64.  Flushed to the global DL at the end
//            with RED.MIN only where the CTA's value beats the global one.
//  smem16  : same with both extremes of a slot packed into one 32-bit word
//            (lo - ybase, 0xFFFF - (hi - ybase)) when the y range spans at
//            most 2^16 values; updates by CAS (rare, filtered).  Twice the
//            columns per CTA, twice the CTAs per SM.
//  global  : any p; the slot table lives in the (L2-resident) global DL,
//            read-compare-then-RED.MIN.
//  filter  : any p; each CTA stages a conservative, quantised snapshot of
//            the DL (per column group, 16-bit bounds) in shared memory and
//            only points outside it touch L2 (read-compare-RED).  A point
//            inside [flo, fhi] of its group cannot change its column: flo is
//            an upper bound of every lo in the group, fhi a lower bound of
//            every hi, and those only move outwards.
//
// Every variant streams the points once with 128-bit non-allocating loads
// (2 points per load, 4 loads in flight per thread) over a persistent grid
// sized from the occupancy calculator.  Out-of-range points are skipped and
// flagged by a min-combined error word (DL[2*width]); the host turns it into
// std::invalid_argument like the reference's validation loop (:175-178).
#include <algorithm>

#include "chp_internal.cuh"

namespace {

constexpr int kThreads = 512;

struct Geo {
    uint32_t base;    // x_off + 1 (mod 2^32): slot = x - base
    uint32_t wcheck;  // slots reachable by an int32 x: min(width, INT_MAX - x_off)
    uint32_t qmax;    // valid y: (uint32)(y - 1) < qmax  (VALIDATE only)
};

// Split the (possibly only 8-byte aligned) point array into an optional
// head point, 16-byte vectors, and an optional tail point.
struct Split {
    uint64_t head;  // 0 or 1 leading scalar point
    uint64_t nvec;  // 16-byte vectors (2 points each)
    bool tail;      // one trailing scalar point at index n-1
};
__host__ __device__ inline Split split_points(const int32_t* xy, uint64_t n) {
    Split s;
    s.head = (n > 0 && (reinterpret_cast<uintptr_t>(xy) & 15)) ? 1 : 0;
    const uint64_t rest = n - s.head;
    s.nvec = rest / 2;
    s.tail = (rest & 1) != 0;
    return s;
}

template <bool VALIDATE>
__device__ __forceinline__ bool accept(const Geo& g, int32_t x, int32_t y, uint32_t& s) {
    s = slot_of(x, g.base);
    bool ok = s < g.wcheck;
    if (VALIDATE) ok = ok && ((uint32_t)y - 1u < g.qmax);
    return ok;
}

__device__ __forceinline__ void flag_error(bool bad, int* DL, uint32_t width) {
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) red_min(DL + 2ull * width, -1);
}

// Streams the points assigned to this thread (grid-stride over vectors,
// unrolled 4x) and calls f(x, y) per point.
template <typename F>
__device__ __forceinline__ void for_each_point(const int32_t* __restrict__ xy, uint64_t n, F&& f) {
    const Split sp = split_points(xy, n);
    const int4* __restrict__ v = reinterpret_cast<const int4*>(xy + 2 * sp.head);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < sp.nvec; i += 4 * stride) {
        const int4 a = ld_stream(v + i);
        const int4 b = ld_stream(v + i + stride);
        const int4 c = ld_stream(v + i + 2 * stride);
        const int4 d = ld_stream(v + i + 3 * stride);
        f(a.x, a.y); f(a.z, a.w);
        f(b.x, b.y); f(b.z, b.w);
        f(c.x, c.y); f(c.z, c.w);
        f(d.x, d.y); f(d.z, d.w);
    }
    for (; i < sp.nvec; i += stride) {
        const int4 a = ld_stream(v + i);
        f(a.x, a.y); f(a.z, a.w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (sp.head) f(xy[0], xy[1]);
        if (sp.tail) f(xy[2 * (n - 1)], xy[2 * (n - 1) + 1]);
    }
}

// ------------------------------------------------------------- DL init
__global__ void k_dl_init(int4* __restrict__ DL4, uint64_t nwords4, int* __restrict__ DL, uint32_t width) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords4; i += stride)
        DL4[i] = make_int4(CHP_EMPTY, CHP_EMPTY, CHP_EMPTY, CHP_EMPTY);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (uint64_t w = nwords4 * 4; w < 2ull * width; ++w) DL[w] = CHP_EMPTY;
        DL[2ull * width] = 0;
        DL[2ull * width + 1] = 0;
    }
}

// ------------------------------------------------------------ smem32
template <bool VALIDATE>
__global__ void __launch_bounds__(kThreads) k_reduce_smem32(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, int* __restrict__ DL) {
    extern __shared__ int2 sL[];
    for (uint32_t c = threadIdx.x; c < width; c += blockDim.x) sL[c] = make_int2(CHP_EMPTY, CHP_EMPTY);
    __syncthreads();
    bool bad = false;
    for_each_point(xy, n, [&](int32_t x, int32_t y) {
        uint32_t s;
        if (!accept<VALIDATE>(g, x, y, s)) {
            bad = true;
            return;
        }
        const int2 e = sL[s];
        if (y < e.x) atomicMin(&sL[s].x, y);
        if (~y < e.y) atomicMin(&sL[s].y, ~y);
    });
    flag_error(bad, DL, width);
    __syncthreads();
    // Flush: only slots where this CTA beats the current global value.
    int2* __restrict__ gL = reinterpret_cast<int2*>(DL);
    for (uint32_t c = threadIdx.x; c < width; c += blockDim.x) {
        const int2 e = sL[c];
        if (e.x == CHP_EMPTY && e.y == CHP_EMPTY) continue;
        const int2 cur = ld_cg2(gL + c);
        if (e.x < cur.x) red_min(DL + 2ull * c, e.x);
        if (e.y < cur.y) red_min(DL + 2ull * c + 1, e.y);
    }
}

// ------------------------------------------------------------ smem16
// Slot word: bits 0-15 a = y - ybase (min), bits 16-31 b = 0xFFFF - a (min).
template <bool VALIDATE>
__global__ void __launch_bounds__(kThreads) k_reduce_smem16(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, int32_t ybase,
                                                            int* __restrict__ DL) {
    extern __shared__ uint32_t sW[];
    for (uint32_t c = threadIdx.x; c < width; c += blockDim.x) sW[c] = 0xFFFFFFFFu;
    __syncthreads();
    bool bad = false;
    for_each_point(xy, n, [&](int32_t x, int32_t y) {
        uint32_t s;
        if (!accept<VALIDATE>(g, x, y, s)) {
            bad = true;
            return;
        }
        const uint32_t a = (uint32_t)y - (uint32_t)ybase;
        if (a > 0xFFFFu) {  // outside the packed window: straight to L2
            red_min(DL + 2ull * s, y);
            red_min(DL + 2ull * s + 1, ~y);
            return;
        }
        const uint32_t b = 0xFFFFu - a;
        uint32_t w = sW[s];
        if (a < (w & 0xFFFFu) || b < (w >> 16)) {
            for (;;) {
                const uint32_t nw = min(w & 0xFFFFu, a) | (min(w >> 16, b) << 16);
                if (nw == w) break;
                const uint32_t old = atomicCAS(&sW[s], w, nw);
                if (old == w) break;
                w = old;
            }
        }
    });
    flag_error(bad, DL, width);
    __syncthreads();
    int2* __restrict__ gL = reinterpret_cast<int2*>(DL);
    for (uint32_t c = threadIdx.x; c < width; c += blockDim.x) {
        const uint32_t w = sW[c];
        const uint32_t a = w & 0xFFFFu, b = w >> 16;
        if (a > 0xFFFFu - b) continue;  // lo > hi: empty
        const int32_t lo = ybase + (int32_t)a;
        const int32_t nhi = ~(ybase + (int32_t)(0xFFFFu - b));
        const int2 cur = ld_cg2(gL + c);
        if (lo < cur.x) red_min(DL + 2ull * c, lo);
        if (nhi < cur.y) red_min(DL + 2ull * c + 1, nhi);
    }
}

// ------------------------------------------------------------ global
template <bool VALIDATE>
__global__ void __launch_bounds__(kThreads) k_reduce_global(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, int* __restrict__ DL) {
    const int2* gL = reinterpret_cast<const int2*>(DL);
    bool bad = false;
    for_each_point(xy, n, [&](int32_t x, int32_t y) {
        uint32_t s;
        if (!accept<VALIDATE>(g, x, y, s)) {
            bad = true;
            return;
        }
        const int2 e = ld_cg2(gL + s);
        if (y < e.x) red_min(DL + 2ull * s, y);
        if (~y < e.y) red_min(DL + 2ull * s + 1, ~y);
    });
    flag_error(bad, DL, width);
}

// ------------------------------------------------------------ filter
// Filter word per group of 2^gshift columns: bits 0-15 fa, 16-31 fb with
//   fa = ceil((max_lo - ybase) / 2^ys),  fb = floor((min_hi - ybase + 1) / 2^ys) - 1,
// and a point is skipped iff fa <= u <= fb for u = (y - ybase) >> ys, which
// implies max_lo <= y <= min_hi ("filter").  Empty / unusable
// groups are 0x0000FFFF (fa = 0xFFFF > fb = 0).
__global__ void k_filter_build(const int* __restrict__ DL, uint32_t width, uint32_t gshift, int32_t ybase,
                               uint32_t ys, uint32_t* __restrict__ F, uint32_t ngroups) {
    const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= ngroups) return;
    const int2* gL = reinterpret_cast<const int2*>(DL);
    const uint32_t c0 = gi << gshift;
    const uint32_t c1 = min(width, c0 + (1u << gshift));
    long long maxlo = LLONG_MIN, minhi = LLONG_MAX;
    bool empty = false;
    for (uint32_t c = c0; c < c1; ++c) {
        const int2 e = ld_cg2(gL + c);
        const long long lo = e.x, hi = ~e.y;
        if (lo > hi) {
            empty = true;
            break;
        }
        maxlo = lo > maxlo ? lo : maxlo;
        minhi = hi < minhi ? hi : minhi;
    }
    uint32_t word = 0x0000FFFFu;
    if (!empty && c0 < c1) {
        const long long q = 1ll << ys;
        long long a = maxlo - ybase;
        long long fa = a <= 0 ? 0 : (a + q - 1) / q;
        long long fb = (minhi - ybase + 1) >= 0 ? (minhi - ybase + 1) / q - 1 : -1;
        if (fb > 0xFFFF) fb = 0xFFFF;
        if (fa <= fb && fa <= 0xFFFF && fb >= 0) word = (uint32_t)fa | ((uint32_t)fb << 16);
    }
    F[gi] = word;
}

template <bool VALIDATE>
__global__ void __launch_bounds__(kThreads) k_reduce_filter(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, uint32_t gshift,
                                                            int32_t ybase, uint32_t ys,
                                                            const uint32_t* __restrict__ F, uint32_t ngroups,
                                                            int* __restrict__ DL) {
    extern __shared__ uint32_t sF[];
    {
        const uint4* F4 = reinterpret_cast<const uint4*>(F);
        uint4* s4 = reinterpret_cast<uint4*>(sF);
        const uint32_t n4 = ngroups / 4;
        for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) s4[i] = __ldcg(F4 + i);
        for (uint32_t i = n4 * 4 + threadIdx.x; i < ngroups; i += blockDim.x) sF[i] = __ldcg(F + i);
    }
    __syncthreads();
    const int2* gL = reinterpret_cast<const int2*>(DL);
    bool bad = false;
    for_each_point(xy, n, [&](int32_t x, int32_t y) {
        uint32_t s;
        if (!accept<VALIDATE>(g, x, y, s)) {
            bad = true;
            return;
        }
        const uint32_t w = sF[s >> gshift];
        const uint32_t u = ((uint32_t)y - (uint32_t)ybase) >> ys;
        // (uint32) y - ybase wraps for y < ybase; then u is huge and fails.
        if ((uint32_t)y - (uint32_t)ybase <= (0xFFFFu << ys | ((1u << ys) - 1u)) && u >= (w & 0xFFFFu) &&
            u <= (w >> 16))
            return;
        const int2 e = ld_cg2(gL + s);
        if (y < e.x) red_min(DL + 2ull * s, y);
        if (~y < e.y) red_min(DL + 2ull * s + 1, ~y);
    });
    flag_error(bad, DL, width);
}

int blocks_for(chp_ctx* ctx, const void* fn, size_t smem, int cap_per_sm) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    if (per_sm > cap_per_sm) per_sm = cap_per_sm;
    return per_sm * ctx->sm_count;
}

}  // namespace

extern "C" uint64_t chp_dl_len(int64_t width) { return width < 1 ? 2 : 2ull * (uint64_t)width + 2; }

extern "C" int chp_dl_init(chp_ctx* ctx, int32_t* d_L, int64_t width) {
    if (!ctx) return CHP_EINVAL;
    if (width < 1 || width > (int64_t)UINT32_MAX / 2) return chp_einval(ctx, "reduce: width must be >= 1");
    const uint64_t words = 2ull * (uint64_t)width;
    const bool aligned = (reinterpret_cast<uintptr_t>(d_L) & 15) == 0;
    const uint64_t n4 = aligned ? words / 4 : 0;
    const int blocks = (int)std::min<uint64_t>((n4 + 255) / 256 + 1, (uint64_t)ctx->sm_count * 8);
    k_dl_init<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<int4*>(d_L), n4, d_L, (uint32_t)width);
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

// Choice of variant: the smallest smem footprint
// that holds the exact table, else the filter path.
extern "C" int chp_reduce(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int64_t width, int64_t q,
                          int64_t x_off, int32_t* d_L, uint32_t flags) {
    if (!ctx) return CHP_EINVAL;
    if (width < 1) return chp_einval(ctx, "reduce: width must be >= 1");
    if (width > (int64_t)INT32_MAX) return chp_einval(ctx, "reduce: width exceeds the int32 slot range");
    if ((reinterpret_cast<uintptr_t>(d_xy) & 7) || (reinterpret_cast<uintptr_t>(d_L) & 7))
        return chp_einval(ctx, "reduce: device buffers must be 8-byte aligned");
    if (x_off + 1 < (int64_t)INT32_MIN || x_off > (int64_t)INT32_MAX)
        return chp_einval(ctx, "reduce: x offset outside the int32 range");
    const bool validate = !(flags & CHP_REDUCE_NO_VALIDATE);
    if (!(flags & CHP_REDUCE_ACCUMULATE)) {
        int rc = chp_dl_init(ctx, d_L, width);
        if (rc) return rc;
    }
    if (n == 0) return CHP_OK;

    Geo g;
    g.base = (uint32_t)(int32_t)(x_off + 1);
    const int64_t reach = (int64_t)INT32_MAX - x_off;  // x <= INT32_MAX
    g.wcheck = (uint32_t)std::min<int64_t>(width, reach);
    g.qmax = q < 0 ? (uint32_t)INT32_MAX : (uint32_t)std::min<int64_t>(q, INT32_MAX);
    const uint32_t w = (uint32_t)width;
    const size_t budget = (size_t)std::min(ctx->smem_optin, 200 * 1024);
    const bool fits32 = (size_t)w * 8 <= budget;
    const bool y16 = validate && q >= 1 && q <= 65536;  // all valid y in [1, 65536]
    const bool fits16 = y16 && (size_t)w * 4 <= budget;

    const bool force_global = flags & CHP_REDUCE_FORCE_GLOBAL;
    const bool force_smem32 = flags & CHP_REDUCE_FORCE_SMEM32;
    const bool force_filter = flags & CHP_REDUCE_FORCE_FILTER;

    if (!force_global && !force_filter && (fits16 && !force_smem32)) {
        const size_t smem = (size_t)w * 4;
        auto fn = validate ? k_reduce_smem16<true> : k_reduce_smem16<false>;
        CHP_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int cap = w >= 8192 ? 2 : 4;
        const int blocks = blocks_for(ctx, (const void*)fn, smem, cap);
        fn<<<blocks, kThreads, smem, ctx->stream>>>(d_xy, n, g, w, 1, d_L);
        CHP_LAUNCHED(ctx);
        ctx->variant = "smem16";
        return CHP_OK;
    }
    if (!force_global && !force_filter && fits32) {
        const size_t smem = (size_t)w * 8;
        auto fn = validate ? k_reduce_smem32<true> : k_reduce_smem32<false>;
        CHP_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int cap = w >= 8192 ? 2 : 4;
        const int blocks = blocks_for(ctx, (const void*)fn, smem, cap);
        fn<<<blocks, kThreads, smem, ctx->stream>>>(d_xy, n, g, w, d_L);
        CHP_LAUNCHED(ctx);
        ctx->variant = "smem32";
        return CHP_OK;
    }
    if (force_filter || (!force_global && q >= 1)) {
        // Filter path: warm-up prefix through L2, snapshot, filtered rest.
        const int64_t yspan = q;  // valid y in [1, q]
        uint32_t ys = 0;
        while ((yspan - 1) >> ys > 0xFFFF) ++ys;
        uint32_t gshift = 0;
        while (((uint64_t)(w + (1u << gshift) - 1) >> gshift) * 4 > budget) ++gshift;
        const uint32_t ngroups = (w + (1u << gshift) - 1) >> gshift;
        int rc = chp_ensure(ctx, ctx->filter, (size_t)ngroups * 4 + 16);
        if (rc) return rc;
        const uint64_t warm = std::min<uint64_t>(n, std::max<uint64_t>(n / 64, (uint64_t)w * 4)) & ~1ull;
        {
            auto fn = validate ? k_reduce_global<true> : k_reduce_global<false>;
            const int blocks = blocks_for(ctx, (const void*)fn, 0, 4);
            if (warm > 0) {
                fn<<<blocks, kThreads, 0, ctx->stream>>>(d_xy, warm, g, w, d_L);
                CHP_LAUNCHED(ctx);
            }
        }
        k_filter_build<<<(ngroups + 255) / 256, 256, 0, ctx->stream>>>(d_L, w, gshift, 1, ys,
                                                                      (uint32_t*)ctx->filter.p, ngroups);
        CHP_LAUNCHED(ctx);
        if (n > warm) {
            const size_t smem = (size_t)ngroups * 4;
            auto fn = validate ? k_reduce_filter<true> : k_reduce_filter<false>;
            CHP_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int blocks = blocks_for(ctx, (const void*)fn, smem, 2);
            fn<<<blocks, kThreads, smem, ctx->stream>>>(d_xy + 2 * warm, n - warm, g, w, gshift, 1, ys,
                                                        (const uint32_t*)ctx->filter.p, ngroups, d_L);
            CHP_LAUNCHED(ctx);
        }
        ctx->variant = "filter";
        return CHP_OK;
    }
    auto fn = validate ? k_reduce_global<true> : k_reduce_global<false>;
    const int blocks = blocks_for(ctx, (const void*)fn, 0, 4);
    fn<<<blocks, kThreads, 0, ctx->stream>>>(d_xy, n, g, w, d_L);
    CHP_LAUNCHED(ctx);
    ctx->variant = "global";
    return CHP_OK;
}

extern "C" int chp_check(chp_ctx* ctx, const int32_t* d_L, int64_t width) {
    if (!ctx) return CHP_EINVAL;
    int32_t err = 0;
    CHP_CUDA(ctx, cudaMemcpyAsync(&err, d_L + 2 * width, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (err != 0) return chp_einval(ctx, "reduce: coordinate out of range");
    return CHP_OK;
}
