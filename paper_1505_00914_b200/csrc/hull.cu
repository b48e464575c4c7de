// hull.cu -- K4: exact convex hull of the reduced set, on device.
//
// Replaces hulls::melkman + canonicalize_hull
// (/root/reference/proj/src/hulls.cpp:137-181, src/geometry.cpp:42-80) for
// chains produced by the reduction.  Melkman's deque is inherently serial
// (53-66 ns per chain point on a CPU core) and, run on the
// north_star order, wrong for single-point columns (F3).  Here the hull is
// built from the two x-monotone sequences K3 emits -- lower = (x, lo) and
// upper = (x, hi) over the valid slots, ascending x, one point per column --
// as two independent lower-hull problems: `lower` as is, and `upper`
// reflected through the origin, (-x, -hi) read back to front, whose lower
// hull is the upper hull rotated by 180 degrees.
//
//   leaf   : one lane per chunk of 32 consecutive points runs the strict
//            monotone chain (pop while cross <= 0); a warp loads its 32
//            chunks together (coalesced) into shared-memory stacks.  A point
//            that is not a strict vertex of its chunk's lower hull lies on or
//            above a segment between two chunk points, so it is no global
//            vertex.
//   merge  : log2(#chunks) levels; one warp merges two x-separated lower
//            hulls A | B by their bridge: i* = first i with
//            Q(i) = [A[i+1] strictly below line A[i] -> tangent(A[i], B)]
//            false (32-ary search across the warp), tangent(q, B) = first j
//            with B[j+1] strictly above line q -> B[j] (binary search per
//            lane; the rightmost touching point, so collinear bridge points
//            drop out).  Result A[0..i*] ++ B[t*..].
//   final  : one CTA stitches lower ++ upper (dropping the shared end
//            points of single-point extreme columns), which is already CCW
//            from the lexicographic minimum; degenerate sets come out as
//            1 or 2 vertices {lexmin, lexmax} as in src/geometry.cpp:29-38.
// With cooperative launch the three stages are ONE kernel (a grid barrier
// per merge level); otherwise one launch per stage and level.
// Orientation tests are exact: 64-bit cross products suffice for these
// inputs (see orient), where the reference needs __int128
// (include/chp/geometry.hpp:29-35).
#include <algorithm>
#include <cstdlib>

#include "chp_internal.cuh"

namespace {

constexpr int kLeaf = 32;

struct P {
    long long x, y;
};

// Exact in 64 bits for K4's inputs: every x lies in one width of at most
// 2^29 slots and every y is an int32, so |dx| < 2^29, |dy| < 2^32 and each
// product is below 2^61 (the reference's __int128 form,
// include/chp/geometry.hpp:29-35, is needed for arbitrary int64 points; the
// 128-bit multiplies doubled the leaf chain's instruction count).
__device__ __forceinline__ int orient(const P& a, const P& b, const P& c) {
    const long long v = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
    return (v > 0) - (v < 0);
}
__device__ __forceinline__ bool peq(const P& a, const P& b) { return a.x == b.x && a.y == b.y; }
__device__ __forceinline__ bool lex_less(const P& a, const P& b) {
    return a.x < b.x || (a.x == b.x && a.y < b.y);
}

// The 32 chunks c0 .. c0+31 of problem `prob`, one per lane of the calling
// warp: the warp loads the chunks' points together (lane l takes point l of
// every chunk, so each load is one contiguous run -- a thread loading its own
// chunk strided the warp's loads 256 bytes apart: 32 sectors per load), then
// each lane runs the strict monotone chain over its chunk in its
// shared-memory stack (kStride entries: the odd stride keeps the lanes'
// stacks on different banks).  The stacks hold the points' int32
// coordinates before the reflection (8 bytes; they always fit), the chain
// works on the reflected 64-bit values.
constexpr int kStride = kLeaf + 1;
__device__ __forceinline__ P from_stack(int2 s, int prob) {
    return prob ? P{-(long long)s.x, -(long long)s.y} : P{s.x, s.y};
}
// Problem 0 is `lower` as is, problem 1 `upper` read back to front (and
// reflected when the points become 64-bit).
__device__ __forceinline__ void leaf_warp(const int2* __restrict__ lower, const int2* __restrict__ upper, long long v,
                                          int prob, uint32_t c0, uint32_t nchunks, uint64_t cap, int2* wstack,
                                          P* __restrict__ buf, int* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const long long base = (long long)c0 * kLeaf;
#pragma unroll
    for (int j0 = 0; j0 < kLeaf; j0 += 8) {
        int2 q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const long long k = base + (long long)(j0 + j) * kLeaf + lane;
            if (k < v) q[j] = prob ? upper[v - 1 - k] : lower[k];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) wstack[(j0 + j) * kStride + lane] = q[j];
    }
    __syncwarp();
    const uint32_t c = c0 + lane;
    if (c < nchunks) {
        const long long b = base + (long long)lane * kLeaf;
        int* cp = cnt + (size_t)prob * nchunks + c;
        if (b >= v) {
            *cp = 0;
        } else {
            int2* stack = wstack + lane * kStride;
            const int m = (int)(min(b + kLeaf, v) - b);
            // the top two entries live in registers
            P t1{0, 0}, t2{0, 0};
            int k = 0;
            for (int i = 0; i < m; ++i) {
                const int2 qs = stack[i];
                const P q = from_stack(qs, prob);
                while (k >= 2 && orient(t2, t1, q) <= 0) {
                    --k;
                    t1 = t2;
                    if (k >= 2) t2 = from_stack(stack[k - 2], prob);
                }
                stack[k++] = qs;
                t2 = t1;
                t1 = q;
            }
            P* out = buf + (size_t)prob * cap + b;
            for (int i = 0; i < k; ++i) out[i] = from_stack(stack[i], prob);
            *cp = k;
        }
    }
    __syncwarp();  // the stacks are reused by the warp's next chunks
}

// First j in [0, nb-1) with orient(q, B[j], B[j+1]) > 0, else nb-1.
__device__ __forceinline__ int tangent(const P& q, const P* B, int nb) {
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (orient(q, B[mid], B[mid + 1]) > 0)
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

// Warp gw (< 2 * npairs, warp-uniform) merges regions 2m and 2m+1 of its
// problem.
// Hulls of up to kStage points in total are first staged in the warp's
// shared-memory slab `wsm` (one coalesced round trip), so the searches'
// dependent loads hit shared memory instead of L2.
constexpr int kStage = 256;
__device__ __forceinline__ void merge_pair(uint32_t gw, int lane, const P* __restrict__ in,
                                           const int* __restrict__ cnt_in, P* __restrict__ out,
                                           int* __restrict__ cnt_out, uint32_t nchunks, uint64_t cap,
                                           uint32_t nregions, uint64_t region_cap, P* wsm) {
    const uint32_t npairs = (nregions + 1) / 2;
    const int prob = gw / npairs;
    const uint32_t m = gw % npairs;
    const uint32_t ra = 2 * m, rb = 2 * m + 1;
    const int na = cnt_in[(size_t)prob * nchunks + ra];
    const int nb = rb < nregions ? cnt_in[(size_t)prob * nchunks + rb] : 0;
    const P* A = in + (size_t)prob * cap + (uint64_t)ra * region_cap;
    const P* B = in + (size_t)prob * cap + (uint64_t)rb * region_cap;
    P* O = out + (size_t)prob * cap + (uint64_t)ra * region_cap;
    int* co = cnt_out + (size_t)prob * nchunks + m;
    if (nb == 0 || na == 0) {
        const P* src = na ? A : B;
        const int ns = na ? na : nb;
        for (int k = lane; k < ns; k += 32) O[k] = src[k];
        if (lane == 0) *co = ns;
        return;
    }
    if (wsm && na + nb <= kStage) {
        for (int k = lane; k < na; k += 32) wsm[k] = A[k];
        for (int k = lane; k < nb; k += 32) wsm[na + k] = B[k];
        __syncwarp();
        A = wsm;
        B = wsm + na;
    }
    // i* = first i in [0, na-1] with Q(i) false; Q(na-1) = false.
    int lo = 0, hi = na - 1;
    while (lo < hi) {
        const int span = hi - lo;
        const int cand = span <= 32 ? lo + lane : lo + (int)(((long long)span * lane) >> 5);
        const bool valid = cand < hi;
        bool q = false;
        if (valid) {
            const int t = tangent(A[cand], B, nb);
            q = orient(A[cand], B[t], A[cand + 1]) < 0;
        }
        const unsigned falses = __ballot_sync(0xffffffffu, valid && !q);
        const unsigned valids = __ballot_sync(0xffffffffu, valid);
        if (span <= 32) {
            lo = hi = falses ? lo + __ffs(falses) - 1 : hi;
            break;
        }
        const int last = 31 - __clz(valids);
        const int c_last = __shfl_sync(0xffffffffu, cand, last);
        if (!falses) {
            lo = c_last + 1;
        } else {
            const int f = __ffs(falses) - 1;
            const int c_f = __shfl_sync(0xffffffffu, cand, f);
            const int c_prev = __shfl_sync(0xffffffffu, cand, f > 0 ? f - 1 : 0);
            hi = c_f;
            if (f > 0) lo = c_prev + 1;
        }
    }
    const int istar = lo;
    const int tstar = tangent(A[istar], B, nb);
    const int keep_a = istar + 1;
    for (int k = lane; k < keep_a; k += 32) O[k] = A[k];
    for (int k = tstar + lane; k < nb; k += 32) O[keep_a + (k - tstar)] = B[k];
    if (lane == 0) *co = keep_a + (nb - tstar);
    __syncwarp();  // the slab is reused by the warp's next pair
}

// The whole CTA: lower ++ reflected upper (dropping the shared end points of
// single-point extreme columns), the axis swap (a reflection, so the order
// reverses for h >= 3), then the rotation to the lexicographic minimum.
// (One thread with a 64-bit modulo per vertex took 314 us at h = 1066.)
__device__ __forceinline__ void final_block(const P* __restrict__ fin, const int* __restrict__ cnt_fin,
                                            uint32_t nchunks, uint64_t cap, const long long* __restrict__ counts,
                                            int swapped, P* __restrict__ tmp, int2* __restrict__ hull,
                                            long long* __restrict__ h_out) {
    __shared__ long long s_best[32];
    if (counts[1] == 0) {
        if (threadIdx.x == 0) *h_out = 0;
        return;
    }
    const P* HL = fin;
    const int nl = cnt_fin[0];
    const P* HU = fin + cap;
    const int nu = cnt_fin[nchunks];
    const P u0{-HU[0].x, -HU[0].y};
    const P ul{-HU[nu - 1].x, -HU[nu - 1].y};
    const int st = peq(u0, HL[nl - 1]) ? 1 : 0;
    const int en = peq(ul, HL[0]) ? nu - 1 : nu;
    const long long h = nl + (long long)(en > st ? en - st : 0);  // (one point: st = 1 > en = 0)
    const bool rev = swapped && h >= 3;
    for (long long k = threadIdx.x; k < h; k += blockDim.x) {
        P q = k < nl ? HL[k] : P{-HU[st + (k - nl)].x, -HU[st + (k - nl)].y};
        if (swapped) q = P{q.y, q.x};
        tmp[rev ? h - 1 - k : k] = q;
    }
    __syncthreads();
    // Lexicographic minimum: (index of the best) per thread, then the block.
    long long best = -1;
    for (long long k = threadIdx.x; k < h; k += blockDim.x)
        if (best < 0 || lex_less(tmp[k], tmp[best])) best = k;
    auto better = [&](long long a, long long b) -> long long {  // -1 = none
        if (a < 0) return b;
        if (b < 0) return a;
        return lex_less(tmp[b], tmp[a]) ? b : a;
    };
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = better(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        best = threadIdx.x < (blockDim.x >> 5) ? s_best[threadIdx.x] : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = better(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (threadIdx.x == 0) s_best[0] = best;
    }
    __syncthreads();
    const long long start = s_best[0];
    for (long long k = threadIdx.x; k < h; k += blockDim.x) {
        long long j = start + k;
        if (j >= h) j -= h;
        const P q = tmp[j];
        hull[k] = make_int2((int)q.x, (int)q.y);
    }
    if (threadIdx.x == 0) *h_out = h;
}

constexpr int kLeafThreads = 128;  // threads per k_hull_leaf CTA (the multi-launch form)
constexpr size_t kLeafSmem = (size_t)kLeafThreads * kStride * sizeof(int2);
constexpr int kCoopThreads = 512;  // every thread of the cooperative form runs leaves
constexpr size_t kCoopSmem = (size_t)kCoopThreads * kStride * sizeof(int2);  // 132 KB
constexpr uint32_t kSmallChunks = 64;  // one-CTA form up to 64 chunks per problem
static_assert((kCoopThreads / 32) * kStage * sizeof(P) <= kCoopSmem, "merge slabs reuse the leaf stacks");

__global__ void __launch_bounds__(kLeafThreads) k_hull_leaf(const int2* __restrict__ lower,
                                                            const int2* __restrict__ upper,
                                                            const long long* __restrict__ counts, uint32_t nchunks,
                                                            uint64_t cap, P* __restrict__ buf,
                                                            int* __restrict__ cnt) {
    extern __shared__ int2 lstacks[];
    const uint32_t c0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    if (c0 >= nchunks) return;
    leaf_warp(lower, upper, counts[1], blockIdx.y, c0, nchunks, cap, lstacks + (threadIdx.x & ~31u) * kStride, buf,
              cnt);
}

__global__ void __launch_bounds__(256) k_hull_merge(const P* __restrict__ in, const int* __restrict__ cnt_in, P* __restrict__ out,
                             int* __restrict__ cnt_out, uint32_t nchunks, uint64_t cap, uint32_t nregions,
                             uint64_t region_cap) {
    __shared__ P slab[256 / 32][kStage];
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= 2 * ((nregions + 1) / 2)) return;
    merge_pair(gw, threadIdx.x & 31, in, cnt_in, out, cnt_out, nchunks, cap, nregions, region_cap,
               slab[threadIdx.x >> 5]);
}

__global__ void k_hull_final(const P* __restrict__ fin, const int* __restrict__ cnt_fin, uint32_t nchunks,
                             uint64_t cap, const long long* __restrict__ counts, int swapped,
                             P* __restrict__ tmp, int2* __restrict__ hull, long long* __restrict__ h_out) {
    final_block(fin, cnt_fin, nchunks, cap, counts, swapped, tmp, hull, h_out);
}

// All of K4 as one cooperative kernel (one CTA per SM): the leaves (every
// thread: a warp takes 32 chunks), a grid barrier per merge level (~1.3 us
// instead of a launch boundary), and the final on CTA 0.  (Rounds of leaf
// filtering with an in-order compaction between them, until few points are
// left, measured slower: ~25 us per round against ~7 us per merge level.)
__global__ void __launch_bounds__(kCoopThreads, 1)
    k_hull_coop(const int2* __restrict__ lower, const int2* __restrict__ upper, const long long* __restrict__ counts,
                uint32_t nchunks, uint64_t cap, P* buf0, P* buf1, int* cnt0, int* cnt1, int swapped, P* tmp,
                int2* __restrict__ hull, long long* __restrict__ h_out, GridBar* bar) {
    extern __shared__ int2 lstacks[];  // leaf stacks; later the merges' slabs
    P* stacks = reinterpret_cast<P*>(lstacks);
    const long long v = counts[1];
    {  // warp tasks: 32 chunks of one problem each
        const uint32_t nwc = (nchunks + 31) / 32;
        const uint32_t lw = threadIdx.x >> 5, nlw = blockDim.x / 32;
        for (uint32_t t = blockIdx.x * nlw + lw; t < 2 * nwc; t += gridDim.x * nlw) {
            const int prob = t >= nwc;
            leaf_warp(lower, upper, v, prob, (prob ? t - nwc : t) * 32, nchunks, cap,
                      lstacks + (threadIdx.x & ~31u) * kStride, buf0, cnt0);
        }
    }
    // (a single CTA -- small widths, launched plainly -- needs no grid barrier)
    if (gridDim.x == 1) __syncthreads(); else grid_barrier(bar);
    P *bin = buf0, *bout = buf1;
    int *cin = cnt0, *cout = cnt1;
    uint32_t nregions = nchunks;
    uint64_t region_cap = kLeaf;
    bool alone = gridDim.x == 1;
    while (nregions > 1) {
        const uint32_t npairs = (nregions + 1) / 2;
        // The last levels (at most one pair per warp of a CTA) on CTA 0
        // alone, with block barriers instead of grid barriers.
        if (!alone && 2 * npairs <= (blockDim.x >> 5)) {
            grid_barrier_done(bar);
            if (blockIdx.x != 0) return;
            alone = true;
        }
        const uint32_t warps = (alone ? 1u : gridDim.x) * (blockDim.x >> 5);
        const uint32_t gw0 = (alone ? 0u : blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
        for (uint32_t gw = gw0; gw < 2 * npairs; gw += warps)
            merge_pair(gw, threadIdx.x & 31, bin, cin, bout, cout, nchunks, cap, nregions, region_cap,
                       stacks + (threadIdx.x >> 5) * kStage);  // the leaf stacks, free after the leaves
        if (alone) __syncthreads(); else grid_barrier(bar);
        P* tb = bin;
        bin = bout;
        bout = tb;
        int* tc = cin;
        cin = cout;
        cout = tc;
        nregions = npairs;
        region_cap *= 2;
    }
    if (!alone) grid_barrier_done(bar);
    if (blockIdx.x == 0) final_block(bin, cin, nchunks, cap, counts, swapped, tmp, hull, h_out);
}

}  // namespace

extern "C" int chp_hull(chp_ctx* ctx, const int32_t* d_lower, const int32_t* d_upper, const int64_t* d_counts,
                        int64_t width, int swapped, int32_t* d_hull, int64_t* d_h) {
    if (!ctx) return CHP_EINVAL;
    if (width < 1 || width > (1ll << 29)) return chp_einval(ctx, "hull: width must be in [1, 2^29]");
    const uint32_t nchunks = (uint32_t)((width + kLeaf - 1) / kLeaf);
    const uint64_t cap = (uint64_t)nchunks * kLeaf;
    int rc;
    if ((rc = chp_ensure(ctx, ctx->hull_a, 2 * cap * sizeof(P) + 2 * (cap + 2) * sizeof(P)))) return rc;
    if ((rc = chp_ensure(ctx, ctx->hull_b, 2 * cap * sizeof(P)))) return rc;
    if ((rc = chp_ensure(ctx, ctx->hull_cnt_a, 2 * (size_t)nchunks * sizeof(int)))) return rc;
    if ((rc = chp_ensure(ctx, ctx->hull_cnt_b, 2 * (size_t)nchunks * sizeof(int)))) return rc;
    P* bufs[2] = {(P*)ctx->hull_a.p, (P*)ctx->hull_b.p};
    int* cnts[2] = {(int*)ctx->hull_cnt_a.p, (int*)ctx->hull_cnt_b.p};
    P* tmp = (P*)ctx->hull_a.p + 2 * cap;
    const long long* counts = reinterpret_cast<const long long*>(d_counts);

    // CHP_HULL_LAUNCHES=1 (tests): the multi-launch form even when the
    // cooperative kernel is available.
    static const bool force_launches = getenv("CHP_HULL_LAUNCHES") != nullptr;
    // Small widths (<= 64 chunks a problem, 2048 columns): the same kernel as
    // ONE CTA, block barriers instead of grid barriers, a plain launch (C5,
    // p = 256: one CTA of 512 threads instead of 148 behind 3 grid barriers).
    if (nchunks <= kSmallChunks && !force_launches) {
        if (!ctx->hull_small_attr) {
            CHP_CUDA(ctx, cudaFuncSetAttribute(k_hull_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kCoopSmem));
            ctx->hull_small_attr = 1;
        }
        k_hull_coop<<<1, kCoopThreads, kCoopSmem, ctx->stream>>>(
            reinterpret_cast<const int2*>(d_lower), reinterpret_cast<const int2*>(d_upper), counts, nchunks, cap,
            bufs[0], bufs[1], cnts[0], cnts[1], swapped, tmp, reinterpret_cast<int2*>(d_hull),
            reinterpret_cast<long long*>(d_h), nullptr);
        CHP_LAUNCHED(ctx);
        return CHP_OK;
    }
    if (ctx->coop && !force_launches) {
        if (!ctx->gridbar.p) {
            if ((rc = chp_ensure(ctx, ctx->gridbar, 64))) return rc;
            CHP_CUDA(ctx, cudaMemsetAsync(ctx->gridbar.p, 0, 64, ctx->stream));
        }
        if (!ctx->hull_coop_checked) {
            ctx->hull_coop_checked = 1;
            int per_sm = 0;
            if (cudaFuncSetAttribute(k_hull_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCoopSmem) ==
                    cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hull_coop, kCoopThreads, kCoopSmem) ==
                    cudaSuccess)
                ctx->hull_coop_ok = per_sm >= 1;
            cudaGetLastError();
        }
        if (ctx->hull_coop_ok) {
            const int2* lo = reinterpret_cast<const int2*>(d_lower);
            const int2* up = reinterpret_cast<const int2*>(d_upper);
            int2* hp = reinterpret_cast<int2*>(d_hull);
            long long* hh = reinterpret_cast<long long*>(d_h);
            GridBar* bar = (GridBar*)ctx->gridbar.p;
            uint32_t nc = nchunks;
            uint64_t cp = cap;
            int sw = swapped;
            void* args[] = {(void*)&lo,      (void*)&up,      (void*)&counts,  (void*)&nc,   (void*)&cp,
                            (void*)&bufs[0], (void*)&bufs[1], (void*)&cnts[0], (void*)&cnts[1], (void*)&sw,
                            (void*)&tmp,     (void*)&hp,      (void*)&hh,      (void*)&bar};
            // (Refused when the grid cannot be co-resident: the launches below.)
            // CHP_TEST_COOP_REFUSE (tests): an oversized grid, which the
            // runtime refuses without running anything.
            static const bool refuse = getenv("CHP_TEST_COOP_REFUSE") != nullptr;
            if (cudaLaunchCooperativeKernel((const void*)k_hull_coop, dim3(ctx->sm_count * (refuse ? 64 : 1)),
                                            dim3(kCoopThreads), args,
                                            kCoopSmem, ctx->stream) == cudaSuccess) {
                CHP_LAUNCHED(ctx);
                return CHP_OK;
            }
            cudaGetLastError();
        }
    }
    if (!ctx->hull_leaf_attr) {
        CHP_CUDA(ctx, cudaFuncSetAttribute(k_hull_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLeafSmem));
        ctx->hull_leaf_attr = 1;
    }
    dim3 lg((nchunks + kLeafThreads - 1) / kLeafThreads, 2);
    k_hull_leaf<<<lg, kLeafThreads, kLeafSmem, ctx->stream>>>(reinterpret_cast<const int2*>(d_lower),
                                                              reinterpret_cast<const int2*>(d_upper), counts,
                                                              nchunks, cap, bufs[0], cnts[0]);
    CHP_LAUNCHED(ctx);
    int cur = 0;
    uint32_t nregions = nchunks;
    uint64_t region_cap = kLeaf;
    while (nregions > 1) {
        const uint32_t npairs = (nregions + 1) / 2;
        const uint64_t threads = 2ull * npairs * 32;
        const int blocks = (int)((threads + 255) / 256);
        k_hull_merge<<<blocks, 256, 0, ctx->stream>>>(bufs[cur], cnts[cur], bufs[cur ^ 1], cnts[cur ^ 1], nchunks,
                                                      cap, nregions, region_cap);
        CHP_LAUNCHED(ctx);
        cur ^= 1;
        nregions = npairs;
        region_cap *= 2;
    }
    k_hull_final<<<1, 1024, 0, ctx->stream>>>(bufs[cur], cnts[cur], nchunks, cap, counts, swapped, tmp,
                                              reinterpret_cast<int2*>(d_hull), reinterpret_cast<long long*>(d_h));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

