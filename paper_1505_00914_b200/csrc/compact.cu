// compact.cu -- K3: skip-invalid compaction of L into the ordered chain.
//
// Replaces build_polyline (/root/reference/proj/src/reducer.cpp:108-119),
// the ctz walk of the occupancy words it iterates
// (include/chp/occupancy.hpp:83-93), ExtremalArray::valid_count
// (src/reducer.cpp:42-49) and serialize's (width+1,-1) form (:121-130).
//
// One pass over the 8-byte slots with a single-pass decoupled look-back scan
// (tiles of 128 threads x 4 or 16 slots, tile order such that every
// predecessor of a tile has started).  The scanned value packs two counters
// in a u64: c = 1 + [hi != lo] per valid slot (chain positions, Lemma-1
// order) in the low word and v = [valid] (lower/upper positions) in the high
// word.  Status words carry a 2-bit flag and both counters in 31 bits each,
// hence width <= 2^29.  A warp of 8-slot masks is folded into 64-bit
// occupancy words with three shuffles (the paper's bit array M, in
// BlockedBitset<uint64_t> layout).
#include <algorithm>

#include "chp_internal.cuh"

namespace {

// 128 threads x ITEMS slots per tile.  ITEMS = 4 (512-slot tiles) up to
// 2^17 slots, so p = 65536 spreads over 128 CTAs (2048-slot tiles left 32
// CTAs latency-bound: 10.5 us at C2); ITEMS = 16 (2048-slot tiles) beyond,
// so the look-back chain of p = 2^20 is 512 tiles long instead of 2048.
constexpr int kCT = 128;  // threads per tile
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

template <int kItems>
__global__ void __launch_bounds__(kCT) k_compact(const int* __restrict__ DL, uint32_t width, Map map,
                                                 int2* __restrict__ chain, unsigned long long* __restrict__ occ,
                                                 int2* __restrict__ lpairs, int2* __restrict__ lower,
                                                 int2* __restrict__ upper, int2* __restrict__ upperd,
                                                 long long* __restrict__ counts,
                                                 unsigned long long* __restrict__ status,
                                                 unsigned long long* __restrict__ status_next, uint32_t ntiles,
                                                 int use_ticket) {
    constexpr int kLanesPerWord = 64 / kItems;
    constexpr int kTile = kCT * kItems;
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_warp[kCT / 32];
    __shared__ unsigned long long s_excl;
    pdl_wait();  // DL from K1 (launched as a programmatic dependent)
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
    // The next call uses the other status array: clear it here instead of a
    // cudaMemset before every launch.
    if (threadIdx.x == 0) {
        status_next[tile] = 0ull;
        if (tile == 0) reinterpret_cast<unsigned int*>(status_next + ntiles)[0] = 0u;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t slot0 = (uint64_t)tile * kTile + (uint64_t)threadIdx.x * kItems;
    const int2* gL = reinterpret_cast<const int2*>(DL);

    int lo[kItems], hi[kItems];
    uint32_t vmask = 0, dmask = 0;
    if (slot0 + kItems <= width && !(reinterpret_cast<uintptr_t>(DL) & 15)) {
        // whole thread in range: 16-byte loads, all in flight together
        const int4* g4 = reinterpret_cast<const int4*>(gL + slot0);
        int4 q[kItems / 2];
#pragma unroll
        for (int j = 0; j < kItems / 2; ++j) q[j] = g4[j];  // (L1: the lane's later loads hit its sectors)
#pragma unroll
        for (int j = 0; j < kItems / 2; ++j) {
            lo[2 * j] = q[j].x;
            hi[2 * j] = ~q[j].y;
            lo[2 * j + 1] = q[j].z;
            hi[2 * j + 1] = ~q[j].w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const uint64_t s = slot0 + j;
            lo[j] = CHP_EMPTY;
            hi[j] = INT_MIN;
            if (s < width) {
                const int2 e = gL[s];
                lo[j] = e.x;
                hi[j] = ~e.y;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        if (lo[j] <= hi[j]) {
            vmask |= 1u << j;
            if (lo[j] != hi[j]) dmask |= 1u << j;
        }
    }
    const uint32_t nv = __popc(vmask), nd = __popc(dmask);
    const unsigned long long mine = (unsigned long long)(nv + nd) | ((unsigned long long)nv << 32);

    // Block exclusive scan of `mine`.
    unsigned long long incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < kCT / 32 ? s_warp[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < kCT / 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        if (lane < kCT / 32) s_warp[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    const unsigned long long warp_excl = warp ? s_warp[warp - 1] : 0ull;
    const unsigned long long tile_agg = s_warp[kCT / 32 - 1];
    const unsigned long long thread_excl = warp_excl + incl - mine;

    // Decoupled look-back (warp 0).
    if (warp == 0) {
        unsigned long long excl = 0;
        if (tile == 0) {
            if (lane == 0) st_release(status + tile, pack_status(kFlagIncl, tile_agg));
        } else {
            if (lane == 0) st_release(status + tile, pack_status(kFlagAgg, tile_agg));
            // Look back over a window of 256 predecessors at once (8 per
            // lane, all loads in flight together): every tile publishes its
            // aggregate right after its local scan, so one window usually
            // settles the prefix in a single L2 round trip instead of a
            // chain of 32-tile steps.  Indices below 0 read as an
            // inclusive zero.
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
                // Re-poll every not-yet-published predecessor together, one
                // round trip per pass (a per-slot spin serialised up to 8
                // L2 round trips per lane: the look-back took ~6 us at C2).
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
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const unsigned long long tile_pre = s_excl;
    const unsigned long long pre = tile_pre + thread_excl;
    const uint32_t C0 = (uint32_t)tile_pre, V0 = (uint32_t)(tile_pre >> 32);  // the tile's first positions
    const uint32_t tileC = (uint32_t)tile_agg, tileV = (uint32_t)(tile_agg >> 32);
    const uint64_t tile_slot0 = (uint64_t)tile * kTile;
    const uint32_t tile_slots = (uint32_t)(width - tile_slot0 < (uint64_t)kTile ? width - tile_slot0 : kTile);

    // Outputs go through a shared-memory stage, one output at a time, and
    // leave the tile as contiguous runs: written straight from registers,
    // each warp store touched 32 sectors for 8 bytes apiece (ncu, C4: 2.1 M
    // store sectors for 16 MB of chain, 31 sectors per request).
    extern __shared__ int2 stage[];  // 2 * kTile points
    auto flush = [&](int2* __restrict__ dst, uint32_t count) {
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < count; k += kCT) dst[k] = stage[k];
        __syncthreads();
    };
    const uint32_t cl = (uint32_t)thread_excl, vl = (uint32_t)(thread_excl >> 32);  // local positions
    if (chain) {
        uint32_t c = cl;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            if (!((vmask >> j) & 1)) continue;
            const long long slot1 = (long long)(slot0 + j) + 1;
            stage[c] = to_original(map, slot1, lo[j]);
            if ((dmask >> j) & 1) stage[c + 1] = to_original(map, slot1, hi[j]);
            c += ((dmask >> j) & 1) ? 2 : 1;
        }
        flush(chain + C0, tileC);
    }
    if (lpairs) {
#pragma unroll
        for (int j = 0; j < kItems; ++j)
            stage[threadIdx.x * kItems + j] =
                ((vmask >> j) & 1) ? make_int2(lo[j], hi[j]) : make_int2((int)(width + 1), -1);
        flush(lpairs + tile_slot0, tile_slots);
    }
    auto stage_side = [&](bool use_hi, bool only_d, uint32_t pos) {
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            if (!((vmask >> j) & 1) || (only_d && !((dmask >> j) & 1))) continue;
            const int32_t major = (int32_t)((long long)(slot0 + j) + 1 + map.major_off);
            stage[pos++] = make_int2(major, (int32_t)((use_hi ? hi[j] : lo[j]) + map.minor_off));
        }
    };
    if (lower) {
        stage_side(false, false, vl);
        flush(lower + V0, tileV);
    }
    if (upper) {
        stage_side(true, false, vl);
        flush(upper + V0, tileV);
    }
    if (upperd) {
        stage_side(true, true, cl - vl);
        flush(upperd + (C0 - V0), tileC - tileV);
    }
    const uint32_t C = (uint32_t)pre + (uint32_t)mine, V = (uint32_t)(pre >> 32) + (uint32_t)(mine >> 32);
    if (occ) {
        // kLanesPerWord lanes x kItems slots = one 64-bit word (the first
        // slot of lane kLanesPerWord*k is 64-aligned).
        unsigned long long word = (unsigned long long)vmask << (kItems * (lane % kLanesPerWord));
#pragma unroll
        for (int o = 1; o < kLanesPerWord; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
        const uint64_t wi = slot0 >> 6;
        if (lane % kLanesPerWord == 0 && wi * 64 < width) occ[wi] = word;
    }
    if (tile == ntiles - 1 && threadIdx.x == kCT - 1) {
        // The last tile's last thread holds the totals.
        counts[0] = (long long)C;
        counts[1] = (long long)V;
        counts[2] = (long long)DL[2ull * width];
        counts[3] = (long long)(C - V);
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
    const uint32_t kTile = kCT * (big ? 16 : 4);
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
    auto kfn = big ? k_compact<16> : k_compact<4>;
    if (ctx->compact_resident == 0) {
        int per_sm = 0, per_sm_big = 0;  // (per-SM limits of the two forms)
        cudaFuncSetAttribute(k_compact<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kCT * 16 * 8);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_compact<4>, kCT, 2 * kCT * 4 * 8);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_big, k_compact<16>, kCT, 2 * kCT * 16 * 8);
        ctx->compact_resident = (uint32_t)std::max(std::min(per_sm, per_sm_big), 1) * (uint32_t)ctx->sm_count;
    }
    const int use_ticket = ntiles > ctx->compact_resident ? 1 : 0;
    Map m{major_off, minor_off, swapped};
    const size_t stage_bytes = 2 * (size_t)kTile * sizeof(int2);
    if (big && !ctx->compact_big_attr) {
        CHP_CUDA(ctx, cudaFuncSetAttribute(k_compact<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)stage_bytes));
        ctx->compact_big_attr = 1;
    }
    CHP_CUDA(ctx, launch_pdl(kfn, dim3(ntiles), dim3(kCT), stage_bytes, ctx->stream, (const int*)d_L, (uint32_t)width, m,
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
