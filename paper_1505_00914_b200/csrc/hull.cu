// hull.cu -- K4: exact convex hull of the reduced set, on device.
//
// Replaces hulls::melkman + canonicalize_hull
// (/root/reference/proj/src/hulls.cpp:396-440, src/geometry.cpp:407-445) for
// chains produced by the reduction.  Melkman's deque is inherently serial
// (53-66 ns per chain point on a CPU core) and, run on the
// north_star order, wrong for single-point columns (F3).  Here the hull is
// built from the two x-monotone sequences K3 emits -- lower = (x, lo) and
// upper = (x, hi) over the valid slots, ascending x, one point per column --
// as two independent lower-hull problems: `lower` as is, and `upper`
// reflected through the origin, (-x, -hi) read back to front, whose lower
// hull is the upper hull rotated by 180 degrees.
//
//   leaf   : one thread per chunk of 32 consecutive points runs the strict
//            monotone chain (pop while cross <= 0).  A point that is not a
//            strict vertex of its chunk's lower hull lies on or above a
//            segment between two chunk points, so it is no global vertex.
//   merge  : log2(#chunks) levels; one warp merges two x-separated lower
//            hulls A | B by their bridge: i* = first i with
//            Q(i) = [A[i+1] strictly below line A[i] -> tangent(A[i], B)]
//            false (32-ary search across the warp), tangent(q, B) = first j
//            with B[j+1] strictly above line q -> B[j] (binary search per
//            lane; the rightmost touching point, so collinear bridge points
//            drop out).  Result A[0..i*] ++ B[t*..].
//   final  : one thread stitches lower ++ upper (dropping the shared end
//            points of single-point extreme columns), which is already CCW
//            from the lexicographic minimum; degenerate sets come out as
//            1 or 2 vertices {lexmin, lexmax} as in src/geometry.cpp:394-403.
// Orientation tests are exact (__int128 cross products,
// include/chp/geometry.hpp:29-35).
#include <algorithm>

#include "chp_internal.cuh"

namespace {

constexpr int kLeaf = 32;

struct P {
    long long x, y;
};

__device__ __forceinline__ int orient(const P& a, const P& b, const P& c) {
    const __int128 v = (__int128)(b.x - a.x) * (c.y - a.y) - (__int128)(b.y - a.y) * (c.x - a.x);
    return (v > 0) - (v < 0);
}
__device__ __forceinline__ bool peq(const P& a, const P& b) { return a.x == b.x && a.y == b.y; }
__device__ __forceinline__ bool lex_less(const P& a, const P& b) {
    return a.x < b.x || (a.x == b.x && a.y < b.y);
}

// Point k of problem `prob`: 0 = lower sequence, 1 = reflected upper.
__device__ __forceinline__ P seq_point(const int2* lower, const int2* upper, long long v, int prob, long long k) {
    if (prob == 0) {
        const int2 q = lower[k];
        return P{q.x, q.y};
    }
    const int2 q = upper[v - 1 - k];
    return P{-(long long)q.x, -(long long)q.y};
}

__global__ void k_hull_leaf(const int2* __restrict__ lower, const int2* __restrict__ upper,
                            const long long* __restrict__ counts, uint32_t nchunks, uint64_t cap,
                            P* __restrict__ buf, int* __restrict__ cnt) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const int prob = blockIdx.y;
    if (c >= nchunks) return;
    const long long v = counts[1];
    const long long b = (long long)c * kLeaf;
    int* cp = cnt + (size_t)prob * nchunks + c;
    if (b >= v) {
        *cp = 0;
        return;
    }
    const long long e = min(b + kLeaf, v);
    P* out = buf + (size_t)prob * cap + b;
    int k = 0;
    for (long long i = b; i < e; ++i) {
        const P q = seq_point(lower, upper, v, prob, i);
        while (k >= 2 && orient(out[k - 2], out[k - 1], q) <= 0) --k;
        out[k++] = q;
    }
    *cp = k;
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

__global__ void k_hull_merge(const P* __restrict__ in, const int* __restrict__ cnt_in, P* __restrict__ out,
                             int* __restrict__ cnt_out, uint32_t nchunks, uint64_t cap, uint32_t nregions,
                             uint64_t region_cap) {
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t npairs = (nregions + 1) / 2;
    if (gw >= 2 * npairs) return;
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
}

__global__ void k_hull_final(const P* __restrict__ fin, const int* __restrict__ cnt_fin, uint32_t nchunks,
                             uint64_t cap, const long long* __restrict__ counts, int swapped,
                             P* __restrict__ tmp, int2* __restrict__ hull, long long* __restrict__ h_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (counts[1] == 0) {
        *h_out = 0;
        return;
    }
    const P* HL = fin;
    const int nl = cnt_fin[0];
    const P* HU = fin + cap;
    const int nu = cnt_fin[nchunks];
    long long h = 0;
    for (int k = 0; k < nl; ++k) tmp[h++] = HL[k];
    const P u0{-HU[0].x, -HU[0].y};
    const P ul{-HU[nu - 1].x, -HU[nu - 1].y};
    const int st = peq(u0, HL[nl - 1]) ? 1 : 0;
    const int en = peq(ul, HL[0]) ? nu - 1 : nu;
    for (int k = st; k < en; ++k) tmp[h++] = P{-HU[k].x, -HU[k].y};
    if (swapped) {
        for (long long k = 0; k < h; ++k) tmp[k] = P{tmp[k].y, tmp[k].x};
        if (h >= 3) {  // a reflection flips the orientation
            for (long long i = 0, j = h - 1; i < j; ++i, --j) {
                const P t = tmp[i];
                tmp[i] = tmp[j];
                tmp[j] = t;
            }
        }
    }
    long long start = 0;
    for (long long k = 1; k < h; ++k)
        if (lex_less(tmp[k], tmp[start])) start = k;
    for (long long k = 0; k < h; ++k) {
        const P q = tmp[(start + k) % h];
        hull[k] = make_int2((int)q.x, (int)q.y);
    }
    *h_out = h;
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

    dim3 lg((nchunks + 127) / 128, 2);
    k_hull_leaf<<<lg, 128, 0, ctx->stream>>>(reinterpret_cast<const int2*>(d_lower),
                                             reinterpret_cast<const int2*>(d_upper), counts, nchunks, cap,
                                             bufs[0], cnts[0]);
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
    k_hull_final<<<1, 32, 0, ctx->stream>>>(bufs[cur], cnts[cur], nchunks, cap, counts, swapped, tmp,
                                            reinterpret_cast<int2*>(d_hull), reinterpret_cast<long long*>(d_h));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}
