// compact.cu -- K3: skip-invalid compaction of L into the ordered chain.
//
// Replaces build_polyline (/root/reference/proj/src/reducer.cpp:108-119),
// the ctz walk of the occupancy words it iterates
// (include/chp/occupancy.hpp:83-93), ExtremalArray::valid_count
// (src/reducer.cpp:42-49) and serialize's (width+1,-1) form (:121-130).
//
// One pass over the 8-byte slots with a single-pass decoupled look-back scan
// (tiles of 256 threads x 4 or 16 slots, striped; tile order such that every
// predecessor of a tile has started).  The scanned value packs two counters
// in a u64: c = 1 + [hi != lo] per valid slot (chain positions, Lemma-1
// order) in the low word and v = [valid] (lower/upper positions) in the high
// word.  Status words carry a 2-bit flag and both counters in 31 bits each,
// hence width <= 2^29.  The occupancy words (the paper's bit array M, in
// BlockedBitset<uint64_t> layout) are warp ballots: two warps' 32 slots per
// 64-bit word.
#include <algorithm>
#include <cstdlib>

#include "chp_internal.cuh"

// Instrumentation build only (CHP_NVCC_EXTRA=-DCHP_K3_TIMING=1): thread 0 of
// every tile stamps %globaltimer at the phase boundaries (chp_debug_k3_phase).
#ifndef CHP_K3_TIMING
#define CHP_K3_TIMING 0
#endif
#if CHP_K3_TIMING
__device__ unsigned long long g_k3_phase[4096][6];
#define K3_MARK(tile, k)                                                              \
    do {                                                                              \
        if (threadIdx.x == 0 && (tile) < 4096) {                                     \
            unsigned long long t_;                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
            g_k3_phase[(tile)][(k)] = t_;                                             \
        }                                                                             \
    } while (0)
#else
#define K3_MARK(tile, k) \
    do {                 \
    } while (0)
#endif

namespace {

// Tiles of 256 threads x 4 slots up to 2^17 slots (p = 65536: 64 CTAs),
// 256 x 16 beyond (p = 2^20: 256 CTAs, so the look-back chain is short).
constexpr uint32_t kSmallTileMax = 1u << 17;

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kMask31 = (1ull << 31) - 1;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, unsigned long long cv) {
    return flag | (cv & kMask31) | (((cv >> 32) & kMask31) << 31);
}
__device__ __forceinline__ unsigned long long unpack_cv(unsigned long long st) {
    return (st & kMask31) | (((st >> 31) & kMask31) << 32);
}
// A status word is self-contained (flag and both counters in one 64-bit
// access) and nothing else is published through it, so relaxed gpu-scope
// accesses suffice; acquire loads cost an L1 invalidate (CCTL.IVALL) each.
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct Map {
    long long major_off, minor_off;
    int swapped;
};
__device__ __forceinline__ int2 to_original(const Map& m, long long slot1, long long value) {
    const int32_t major = (int32_t)(slot1 + m.major_off);
    const int32_t minor = (int32_t)(value + m.minor_off);
    return m.swapped ? make_int2(minor, major) : make_int2(major, minor);
}

// Decoupled look-back by warp 0 of a tile: publishes the tile's aggregate,
// returns the exclusive prefix of all preceding tiles (every lane), and
// publishes the inclusive value.  Looks back over a window of 256
// predecessors at once (8 per lane, all loads in flight together): every tile
// publishes its aggregate right after its local scan, so one window usually
// settles the prefix in a single L2 round trip instead of a chain of 32-tile
// steps.  Indices below 0 read as an inclusive zero.
__device__ __forceinline__ unsigned long long lookback(unsigned long long* __restrict__ status, uint32_t tile,
                                                       unsigned long long tile_agg, int lane) {
    unsigned long long excl = 0;
    if (tile == 0) {
        if (lane == 0) st_release(status + tile, pack_status(kFlagIncl, tile_agg));
        return 0;
    }
    if (lane == 0) st_release(status + tile, pack_status(kFlagAgg, tile_agg));
    constexpr int kPer = 8;
    long long top = (long long)tile - 1;
    for (;;) {
        unsigned long long st[kPer];
        long long idx[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            idx[k] = top - lane - 32 * k;
            st[k] = idx[k] >= 0 ? ld_acquire(status + idx[k]) : kFlagIncl;
        }
        // Re-poll every not-yet-published predecessor together, one round
        // trip per pass (a per-slot spin serialised up to 8 L2 round trips
        // per lane: the look-back took ~6 us at C2).
        for (;;) {
            uint32_t pending = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) pending |= (uint32_t)((st[k] >> 62) == 0) << k;
            if (!__any_sync(0xffffffffu, pending != 0)) break;
#pragma unroll
            for (int k = 0; k < kPer; ++k)
                if ((pending >> k) & 1) st[k] = ld_acquire(status + idx[k]);
        }
        long long best = LLONG_MIN;  // nearest inclusive predecessor in the window
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if ((st[k] >> 62) == 2 && idx[k] > best) best = idx[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long b = __shfl_xor_sync(0xffffffffu, best, o);
            best = b > best ? b : best;
        }
        unsigned long long val = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (idx[k] >= best && idx[k] >= 0) val += unpack_cv(st[k]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (best != LLONG_MIN) break;
        top -= 32 * kPer;
    }
    if (lane == 0) st_release(status + tile, pack_status(kFlagIncl, excl + tile_agg));
    return excl;
}

// One tile = kCT threads x kItems slots, STRIPED: item j of thread t is slot
// tile_slot0 + j * kCT + t, so every load of L, and every store of each
// output, is a warp-contiguous run (a blocked layout -- each thread owning
// kItems consecutive slots -- needed a shared-memory stage whose scattered
// writes were 32-way bank conflicts: 8 us of a 20 us call at p = 2^20).
// Chain positions follow slot order, i.e. (item, warp, lane) order: a warp
// scan per item, the (item, warp) totals prefix-summed once in shared memory,
// then the tile's look-back prefix.  Counters per value: c = 1 + [hi != lo]
// (chain) in bits 0-15 and v = [valid] in bits 16-31 (tile-local sums stay
// below 2^16).
template <int kCT, int kItems>
__global__ void __launch_bounds__(kCT) k_compact(const int* __restrict__ DL, uint32_t width, Map map,
                                                 int2* __restrict__ chain, unsigned long long* __restrict__ occ,
                                                 int2* __restrict__ lpairs, int2* __restrict__ lower,
                                                 int2* __restrict__ upper, int2* __restrict__ upperd,
                                                 long long* __restrict__ counts,
                                                 unsigned long long* __restrict__ status,
                                                 unsigned long long* __restrict__ status_next, uint32_t ntiles,
                                                 int use_ticket) {
    static_assert(kCT % 64 == 0, "a warp pair must cover whole 64-bit occupancy words");
    constexpr int kWarps = kCT / 32;
    constexpr int kTile = kCT * kItems;
    static_assert(2 * kTile < 65536, "tile-local counters are 16-bit");
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_tot[kItems * kWarps];  // per (item, warp): c | v << 16, then its exclusive prefix
    __shared__ unsigned long long s_excl, s_agg;
    pdl_wait();  // DL from K1 (launched as a programmatic dependent)
    // (No early trigger here: a caller may reduce K3's own chain next, and
    // the kernels that stream points before their wait rely on their
    // immediate predecessor never writing points.)
    // Tile order: block index when every tile's CTA is co-resident (no
    // predecessor can be waiting for a slot), else an atomic ticket so that
    // a tile only starts after all its predecessors have.
    uint32_t tile = blockIdx.x;
    if (use_ticket) {
        unsigned int* tile_counter = reinterpret_cast<unsigned int*>(status + ntiles);
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        tile = s_tile;
    }
    K3_MARK(tile, 0);
    // The next call uses the other status array: clear it here instead of a
    // cudaMemset before every launch.
    if (threadIdx.x == 0) {
        status_next[tile] = 0ull;
        if (tile == 0) reinterpret_cast<unsigned int*>(status_next + ntiles)[0] = 0u;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t tile_slot0 = (uint64_t)tile * kTile;
    const int2* gL = reinterpret_cast<const int2*>(DL);

    int lo[kItems], hi[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {  // all loads in flight together
        const uint64_t s = tile_slot0 + (uint64_t)j * kCT + threadIdx.x;
        int2 e = make_int2(CHP_EMPTY, CHP_EMPTY);
        if (s < width) e = __ldcg(gL + s);
        lo[j] = e.x;
        hi[j] = ~e.y;
    }
    uint32_t ex[kItems];  // lane-exclusive (c | v << 16) within the warp, per item
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const bool v = lo[j] <= hi[j];
        const uint32_t mine = v ? (lo[j] != hi[j] ? 2u : 1u) | (1u << 16) : 0u;
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        ex[j] = incl - mine;
        if (lane == 31) s_tot[j * kWarps + warp] = incl;
    }
    __syncthreads();
    if (warp == 0) {
        // exclusive prefix over the kItems * kWarps (item, warp) totals, in order
        constexpr int kN = kItems * kWarps;
        constexpr int kPerLane = (kN + 31) / 32;
        uint32_t t[kPerLane], sum = 0;
#pragma unroll
        for (int k = 0; k < kPerLane; ++k) {
            const int i = lane * kPerLane + k;
            t[k] = i < kN ? s_tot[i] : 0u;
            sum += t[k];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        uint32_t run = incl - sum;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kPerLane; ++k) {
            const int i = lane * kPerLane + k;
            if (i < kN) s_tot[i] = run;
            run += t[k];
        }
        K3_MARK(tile, 1);
        const unsigned long long agg = (unsigned long long)(total & 0xFFFFu) | ((unsigned long long)(total >> 16) << 32);
        const unsigned long long excl = lookback(status, tile, agg, lane);
        if (lane == 0) {
            s_excl = excl;
            s_agg = agg;
        }
    }
    __syncthreads();
    K3_MARK(tile, 2);
    const unsigned long long tile_pre = s_excl;
    const uint32_t C0 = (uint32_t)tile_pre, V0 = (uint32_t)(tile_pre >> 32);
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const uint64_t s = tile_slot0 + (uint64_t)j * kCT + threadIdx.x;
        const bool v = lo[j] <= hi[j], d = v && lo[j] != hi[j];
        const uint32_t pre = s_tot[j * kWarps + warp] + ex[j];
        const uint32_t C = C0 + (pre & 0xFFFFu), V = V0 + (pre >> 16);
        CHP_CHECK(!v || s < width);
        CHP_CHECK(!v || C + (d ? 1u : 0u) < 2u * width);
        CHP_CHECK(!v || V < width);
        if (lpairs && s < width) lpairs[s] = v ? make_int2(lo[j], hi[j]) : make_int2((int)(width + 1), -1);
        if (occ) {
            // warps 2k and 2k+1 of an item cover one 64-slot word: its halves
            const uint32_t bits = __ballot_sync(0xffffffffu, v);
            const uint64_t s0 = tile_slot0 + (uint64_t)j * kCT + (uint64_t)warp * 32;
            CHP_CHECK((s0 & 31) == 0);
            if (lane == 0 && (s0 >> 6) < ((uint64_t)width + 63) / 64)  // (the word exists)
                reinterpret_cast<uint32_t*>(occ)[s0 >> 5] = bits;
        }
        if (!v) continue;
        const long long slot1 = (long long)s + 1;
        if (chain) {
            chain[C] = to_original(map, slot1, lo[j]);
            if (d) chain[C + 1] = to_original(map, slot1, hi[j]);
        }
        const int32_t major = (int32_t)(slot1 + map.major_off);
        if (lower) lower[V] = make_int2(major, (int32_t)(lo[j] + map.minor_off));
        if (upper) upper[V] = make_int2(major, (int32_t)(hi[j] + map.minor_off));
        if (upperd && d) upperd[C - V] = make_int2(major, (int32_t)(hi[j] + map.minor_off));
    }
    K3_MARK(tile, 3);
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        const unsigned long long tot = tile_pre + s_agg;
        CHP_CHECK((uint32_t)tot <= 2u * width && (uint32_t)(tot >> 32) <= width);
        counts[0] = (long long)(uint32_t)tot;
        counts[1] = (long long)(uint32_t)(tot >> 32);
        counts[2] = (long long)DL[2ull * width];
        counts[3] = (long long)((uint32_t)tot - (uint32_t)(tot >> 32));
    }
}

__global__ void k_ns_chain(const int2* __restrict__ lower, const int2* __restrict__ upperd,
                           const long long* __restrict__ counts, uint64_t cap, int2* __restrict__ ns) {
    const long long s = counts[0], v = counts[1], d = counts[3];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cap && (long long)k < s; k += stride)
        ns[k] = (long long)k < v ? lower[k] : upperd[d - 1 - ((long long)k - v)];
}

}  // namespace

extern "C" int chp_compact(chp_ctx* ctx, const int32_t* d_L, int64_t width, int64_t major_off,
                           int64_t minor_off, int swapped, int32_t* d_chain, uint64_t* d_occ,
                           int32_t* d_Lpairs, int32_t* d_lower, int32_t* d_upper, int32_t* d_upperd,
                           int64_t* d_counts) {
    if (!ctx) return CHP_EINVAL;
    if (width < 1 || width > (1ll << 29)) return chp_einval(ctx, "compact: width must be in [1, 2^29]");
    if (!d_counts) return chp_einval(ctx, "compact: counts buffer required");
    const bool big = (uint64_t)width > kSmallTileMax;
    // Tile shape (threads x slots per thread): 256 x 4 up to 2^17 slots,
    // 256 x 16 beyond (CHP_K3_SMALL / CHP_K3_BIG pick others, experiments).
    // Measured alone (tools/k3_bench.py) -- C2, p = 2^16: 128x4 3.5, 256x4 3.3,
    // 256x2 3.7, 128x8 3.8, 64x8 4.2 us; C4, p = 2^20: 256x16 9.3, 128x16
    // 13.6, 256x8 14.1, 512x4 13.9, 128x8 15.0 us.
    static const int small_form = getenv("CHP_K3_SMALL") ? atoi(getenv("CHP_K3_SMALL")) : 5;
    static const int big_form = getenv("CHP_K3_BIG") ? atoi(getenv("CHP_K3_BIG")) : 1;
    static const int forms[][2] = {{128, 4}, {256, 16}, {256, 8}, {512, 4}, {128, 8}, {256, 4}, {64, 8}, {256, 2},
                                   {128, 16}};
    const int f = big ? big_form : small_form;
    const int fi = f >= 0 && f < 9 ? f : 0;
    int thr = forms[fi][0], items = forms[fi][1];
    const uint32_t kTile = (uint32_t)(thr * items);
    const uint32_t ntiles = (uint32_t)((width + kTile - 1) / kTile);
    // Two status arrays of (cap + 2) words, used alternately; each launch
    // clears the other one's first ntiles entries (no memset per call).
    const size_t need = 2 * ((size_t)ntiles + 2) * 8;
    if (ctx->tile_status.bytes < need) {
        int rc = chp_ensure(ctx, ctx->tile_status, need);
        if (rc) return rc;
        ctx->status_cap = (uint32_t)(ctx->tile_status.bytes / 16 - 2);
        CHP_CUDA(ctx, cudaMemsetAsync(ctx->tile_status.p, 0, ctx->tile_status.bytes, ctx->stream));
        ctx->status_clean[0] = ctx->status_clean[1] = ctx->status_cap;
    }
    unsigned long long* base = reinterpret_cast<unsigned long long*>(ctx->tile_status.p);
    const int cur = ctx->status_parity;
    unsigned long long* st_cur = base + (size_t)cur * (ctx->status_cap + 2);
    unsigned long long* st_next = base + (size_t)(cur ^ 1) * (ctx->status_cap + 2);
    if (ctx->status_clean[cur] < ntiles)
        CHP_CUDA(ctx, cudaMemsetAsync(st_cur, 0, ((size_t)ctx->status_cap + 2) * 8, ctx->stream));
    decltype(&k_compact<128, 4>) kfn = k_compact<128, 4>;
    if (thr == 256 && items == 16) kfn = k_compact<256, 16>;
    if (thr == 256 && items == 8) kfn = k_compact<256, 8>;
    if (thr == 512 && items == 4) kfn = k_compact<512, 4>;
    if (thr == 128 && items == 8) kfn = k_compact<128, 8>;
    if (thr == 256 && items == 4) kfn = k_compact<256, 4>;
    if (thr == 64 && items == 8) kfn = k_compact<64, 8>;
    if (thr == 256 && items == 2) kfn = k_compact<256, 2>;
    if (thr == 128 && items == 16) kfn = k_compact<128, 16>;
    if (ctx->compact_resident == 0 || ctx->compact_form != thr * 64 + items) {
        int per_sm = 0;
        CHP_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kfn, thr, 0));
        ctx->compact_resident = (uint32_t)std::max(per_sm, 1) * (uint32_t)ctx->sm_count;
        ctx->compact_form = thr * 64 + items;
    }
    const int use_ticket = ntiles > ctx->compact_resident ? 1 : 0;
    Map m{major_off, minor_off, swapped};
    CHP_CUDA(ctx, launch_pdl(kfn, dim3(ntiles), dim3(thr), 0, ctx->stream, (const int*)d_L, (uint32_t)width, m,
                             reinterpret_cast<int2*>(d_chain), reinterpret_cast<unsigned long long*>(d_occ),
                             reinterpret_cast<int2*>(d_Lpairs), reinterpret_cast<int2*>(d_lower),
                             reinterpret_cast<int2*>(d_upper), reinterpret_cast<int2*>(d_upperd),
                             reinterpret_cast<long long*>(d_counts), st_cur, st_next, ntiles, use_ticket));
    CHP_LAUNCHED(ctx);
    ctx->status_clean[cur] = 0;         // dirty now
    ctx->status_clean[cur ^ 1] = ntiles;  // cleared by this launch
    ctx->status_parity = cur ^ 1;
    return CHP_OK;
}

#if CHP_K3_TIMING
extern "C" int chp_debug_k3_phase(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_k3_phase, sizeof(g_k3_phase));
}
#endif

extern "C" int chp_ns_chain(chp_ctx* ctx, const int32_t* d_lower, const int32_t* d_upperd,
                            const int64_t* d_counts, int64_t width, int32_t* d_ns) {
    if (!ctx) return CHP_EINVAL;
    if (width < 1) return chp_einval(ctx, "ns_chain: width must be >= 1");
    const uint64_t cap = 2ull * (uint64_t)width;
    const int blocks = (int)std::min<uint64_t>((cap + 255) / 256, (uint64_t)ctx->sm_count * 16);
    k_ns_chain<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const int2*>(d_lower),
                                                reinterpret_cast<const int2*>(d_upperd),
                                                reinterpret_cast<const long long*>(d_counts), cap,
                                                reinterpret_cast<int2*>(d_ns));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}
