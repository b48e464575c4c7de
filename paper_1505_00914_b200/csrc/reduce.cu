// reduce.cu -- K1: Algorithm 1 (per-x-column min/max of y) on sm_100a.
//
// Replaces reducer::reduce's validation pass and the bucket() fold
// (/root/reference/proj/src/reducer.cpp:69-79, :19-32).  The fold is a
// scatter-min over a p-slot table, so the kernel is HBM-bound on the 8-byte
// point stream when every per-point table access stays on chip:
//
//  smem32  : slot table privatised per CTA in shared memory, 8 B per slot
//            (lo, ~hi); read-compare-then-ATOMS, so a point that changes
//            nothing costs one LDS.64.  Flushed to the global DL at the end
//            with RED.MIN only where the CTA's value beats the global one.
//  smem16  : both extremes of a slot packed into one 32-bit word
//            (y-1, 0xFFFF-(y-1)) minima when 1 <= y <= q <= 2^16; the hit
//            test is one VIMNMX.U16x2, updates by CAS (rare).
//  sampled : mid-size p: a per-column 8-bit strict-interior filter learned
//            from an n/8 sample (racy per-CTA tables, byte-wise min merge),
//            then one pass over all points; a miss REDs one side.
//  filter  : any p; each CTA stages a conservative, quantised snapshot of
//            the DL per column group in shared memory, rebuilt between
//            phases of doubling length; only points outside it touch L2
//            (read-compare-RED while the snapshots are young, one-sided RED
//            after).  A point inside [flo, fhi] of its group cannot change
//            its column: flo bounds every lo in the group from above, fhi
//            every hi from below, and those only move outwards.
//  global  : any p, no y bound; the slot table lives in the (L2-resident)
//            global DL, read-compare-then-RED.MIN.
//
// Every variant streams the points once with 128-bit non-allocating loads
// (2 points per load, software-pipelined) over a persistent grid sized from
// the occupancy calculator.  Out-of-range points are flagged by a
// min-combined error word (DL[2*width]); the host turns it into
// std::invalid_argument like the reference's validation loop (:175-178).
// In sampled/filter the validation is folded into the miss path (DESIGN.md
// §3); smem16 checks each point branch-free (two compares, a select).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "chp_internal.cuh"
#include "stream.cuh"

namespace {

constexpr int kThreads = 1024;

// Instrumentation build only (CHP_NVCC_EXTRA=-DCHP_PHASE_TIMING=1, read by
// tools/phase_timing.py): thread 0 of every CTA stamps %globaltimer at the
// sampled pipeline's phase boundaries.
#ifndef CHP_PHASE_TIMING
#define CHP_PHASE_TIMING 0
#endif
#if CHP_PHASE_TIMING
__device__ unsigned long long g_phase[160][8];
__device__ __forceinline__ void phase_mark(int k) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_phase[blockIdx.x][k] = t;
    }
}
#else
__device__ __forceinline__ void phase_mark(int) {}
#endif

struct Geo {
    uint32_t base;    // x_off + 1 (mod 2^32): slot = x - base
    uint32_t wcheck;  // slots reachable by an int32 x: min(width, INT_MAX - x_off)
    uint32_t ybase;   // lowest valid y (1 for reduce; the bbox minimum for precondition)
    uint32_t qmax;    // valid y: (uint32)(y - ybase) < qmax  (VALIDATE only)
    uint32_t blocked; // register stream: per-CTA contiguous slices (1) or grid-stride (0)
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
    if (VALIDATE) ok = ok && ((uint32_t)y - g.ybase < g.qmax);
    return ok;
}

// An opaque copy: the value must live in a register from here on, so the
// compiler cannot rematerialise it (uniform-datapath S2UR/LDCU) per use.
__device__ __forceinline__ uint32_t pin(uint32_t v) {
    asm volatile("" : "+r"(v));
    return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void flag_error(bool bad, int* DL, uint32_t width) {
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) red_min(DL + 2ull * width, -1);
}

// Streams the points assigned to this thread (grid-stride over 16-byte
// vectors, 4 vectors per group) and calls f(x, y) per point.  Software
// pipelined: the 4 loads of group k+1 are issued before group k is
// processed, so 8 x 16 B per thread are in flight while the table is
// updated and DRAM latency overlaps the per-point work.
template <typename G, typename F>
__device__ __forceinline__ void for_each_group(const int32_t* __restrict__ xy, uint64_t n, G&& g8, F&& f,
                                               bool blocked = false) {
    const Split sp = split_points(xy, n);
    const int4* __restrict__ v = reinterpret_cast<const int4*>(xy + 2 * sp.head);
    // Grid-stride, or (blocked) each CTA streams its own contiguous slice.
    const uint64_t stride = blocked ? blockDim.x : (uint64_t)gridDim.x * blockDim.x;
    const uint64_t end = blocked ? sp.nvec * (blockIdx.x + 1) / gridDim.x : sp.nvec;
    uint64_t i = (blocked ? sp.nvec * blockIdx.x / gridDim.x : (uint64_t)blockIdx.x * blockDim.x) + threadIdx.x;
    // Trip counts are warp-uniform (tested on the warp's last lane), so the
    // full-mask __syncwarp below is always matched.
    const uint64_t last = 31 - (threadIdx.x & 31);
    if (i + last + 3 * stride < end) {
        // (A ping-pong variant without the register copies below measured
        // 2x slower for smem16 on B200 -- kept simple.)
        int4 a = ld_stream(v + i), b = ld_stream(v + i + stride);
        int4 c = ld_stream(v + i + 2 * stride), d = ld_stream(v + i + 3 * stride);
        for (;;) {
            const uint64_t nx = i + 4 * stride;
            const bool more = nx + last + 3 * stride < end;
            int4 a2, b2, c2, d2;
            if (more) {
                a2 = ld_stream(v + nx);
                b2 = ld_stream(v + nx + stride);
                c2 = ld_stream(v + nx + 2 * stride);
                d2 = ld_stream(v + nx + 3 * stride);
            }
            g8(a, b, c, d);
            // Reconverge: a lane that took an update path (CAS loop, L2
            // miss) must not leave the warp split for the rest of the
            // stream, or every later load and compare is issued once per
            // lane group (ncu: 13.7x instructions, 5.5x DRAM re-reads).
            __syncwarp();
            i = nx;
            if (!more) break;
            a = a2; b = b2; c = c2; d = d2;
        }
    }
    for (; i < end; i += stride) {
        const int4 a = ld_stream(v + i);
        f(a.x, a.y); f(a.z, a.w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (sp.head) f(xy[0], xy[1]);
        if (sp.tail) f(xy[2 * (n - 1)], xy[2 * (n - 1) + 1]);
    }
}

// Ping-pong form of the same loop: two register sets alternate, so no
// per-group register copies.  Measured per kernel: +8% for the sampled
// filter (C2), -50% for smem16 (C3/C5), so only k_reduce_sampled uses it.
template <typename G8, typename F>
__device__ __forceinline__ void for_each_group_pp(const int32_t* __restrict__ xy, uint64_t n, G8&& g8, F&& f) {
    const Split sp = split_points(xy, n);
    const int4* __restrict__ v = reinterpret_cast<const int4*>(xy + 2 * sp.head);
    // Each CTA streams its own contiguous slice (C2's sampled main pass:
    // 596-601 vs 586-587 Gpts/s for grid-stride).
    const uint64_t stride = blockDim.x;
    const uint64_t vb = sp.nvec * blockIdx.x / gridDim.x, ve = sp.nvec * (blockIdx.x + 1) / gridDim.x;
    uint64_t i = vb + threadIdx.x;
    const uint64_t last = 31 - (threadIdx.x & 31);
    if (i + last + 3 * stride < ve) {
        int4 a = ld_stream(v + i), b = ld_stream(v + i + stride);
        int4 c = ld_stream(v + i + 2 * stride), d = ld_stream(v + i + 3 * stride);
        int4 a2, b2, c2, d2;
        for (;;) {
            uint64_t nx = i + 4 * stride;
            bool more = nx + last + 3 * stride < ve;
            if (more) {
                a2 = ld_stream(v + nx);
                b2 = ld_stream(v + nx + stride);
                c2 = ld_stream(v + nx + 2 * stride);
                d2 = ld_stream(v + nx + 3 * stride);
            }
            g8(a, b, c, d);
            __syncwarp();
            i = nx;
            if (!more) break;
            nx = i + 4 * stride;
            more = nx + last + 3 * stride < ve;
            if (more) {
                a = ld_stream(v + nx);
                b = ld_stream(v + nx + stride);
                c = ld_stream(v + nx + 2 * stride);
                d = ld_stream(v + nx + 3 * stride);
            }
            g8(a2, b2, c2, d2);
            __syncwarp();
            i = nx;
            if (!more) break;
        }
    }
    for (; i < ve; i += stride) {
        const int4 a = ld_stream(v + i);
        f(a.x, a.y);
        f(a.z, a.w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (sp.head) f(xy[0], xy[1]);
        if (sp.tail) f(xy[2 * (n - 1)], xy[2 * (n - 1) + 1]);
    }
}


// Per-point form: the 8 points of a group are processed one after another.
template <typename F>
__device__ __forceinline__ void for_each_point(const int32_t* __restrict__ xy, uint64_t n, F&& f) {
    for_each_group(
        xy, n,
        [&](const int4& a, const int4& b, const int4& c, const int4& d) {
            f(a.x, a.y); f(a.z, a.w);
            f(b.x, b.y); f(b.z, b.w);
            f(c.x, c.y); f(c.z, c.w);
            f(d.x, d.y); f(d.z, d.w);
        },
        f);
}

// Batched L2 path for the points of a group that the on-chip table could
// not settle (bit k of `miss`): all their slot loads are issued before any
// compare, so a thread waits for one L2 round trip per group instead of one
// per miss.  READ_FIRST = false skips the loads and REDs both extremes
// (fire-and-forget; right when most misses are real updates).
template <bool READ_FIRST, int N>
__device__ __forceinline__ void settle_misses(uint32_t miss, const uint32_t (&s)[N], const int (&y)[N],
                                              int* __restrict__ DL) {
    if (!miss) return;
#pragma unroll
    for (int k = 0; k < N; ++k) CHP_CHECK(!((miss >> k) & 1) || s[k] < 0x7FFFFFFFu);
    const int2* gL = reinterpret_cast<const int2*>(DL);
    if (READ_FIRST) {
        int2 e[N];
#pragma unroll
        for (int k = 0; k < N; ++k)
            if ((miss >> k) & 1) e[k] = ld_cg2(gL + s[k]);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (!((miss >> k) & 1)) continue;
            if (y[k] < e[k].x) red_min(DL + 2ull * s[k], y[k]);
            if (~y[k] < e[k].y) red_min(DL + 2ull * s[k] + 1, ~y[k]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if (!((miss >> k) & 1)) continue;
            red_min(DL + 2ull * s[k], y[k]);
            red_min(DL + 2ull * s[k] + 1, ~y[k]);
        }
    }
}

__device__ __forceinline__ void unpack4(const int4& a, const int4& b, int (&x)[4], int (&y)[4]) {
    x[0] = a.x; y[0] = a.y; x[1] = a.z; y[1] = a.w;
    x[2] = b.x; y[2] = b.y; x[3] = b.z; y[3] = b.w;
}

// The point stream of one kernel: TMA ring (TMA = true; `ring` points at the
// ring's shared memory) or software-pipelined registers.  g4(a, b) gets four
// points at a time, f(x, y) single points (remainders).
template <bool TMA, typename G4, typename F>
__device__ __forceinline__ void stream_points(const int32_t* __restrict__ xy, uint64_t n, uint8_t* ring,
                                              int stages, G4&& g4, F&& f, bool blocked = false) {
    if (TMA) {
        const Split sp = split_points(xy, n);
        const int4* v = reinterpret_cast<const int4*>(xy + 2 * sp.head);
        chpstream::tma_stream(v, sp.nvec, chpstream::ring_at(ring, stages), g4, [&](const int4& a) {
            f(a.x, a.y);
            f(a.z, a.w);
        });
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (sp.head) f(xy[0], xy[1]);
            if (sp.tail) f(xy[2 * (n - 1)], xy[2 * (n - 1) + 1]);
        }
    } else {
        for_each_group(
            xy, n,
            [&](const int4& a, const int4& b, const int4& c, const int4& d) {
                g4(a, b);
                g4(c, d);
            },
            f, blocked);
    }
}

// Four calls of a per-point functor.
template <typename F>
__device__ __forceinline__ auto per_point4(F& f) {
    return [&f](const int4& a, const int4& b) {
        f(a.x, a.y); f(a.z, a.w);
        f(b.x, b.y); f(b.z, b.w);
    };
}

// Dynamic shared memory: [table, 128-byte aligned][TMA ring].
__host__ __device__ constexpr size_t table_span(size_t table_bytes) { return (table_bytes + 127) & ~(size_t)127; }

// ------------------------------------------------------------- DL init
__global__ void k_dl_init(int4* __restrict__ DL4, uint64_t nwords4, int* __restrict__ DL, uint32_t width) {
    // A programmatic dependent itself (the previous call's K3 reads DL), and
    // the trigger comes after the wait: K1, which streams its points before
    // waiting, may then overlap this grid only, never a kernel before it.
    pdl_wait();
    pdl_trigger();
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
template <bool VALIDATE, bool TMA>
__global__ void __launch_bounds__(kThreads) k_reduce_smem32(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, int stages,
                                                            int* __restrict__ DL) {
    extern __shared__ uint4 smem4[];
    int2* sL = reinterpret_cast<int2*>(smem4);
    uint8_t* ring = reinterpret_cast<uint8_t*>(smem4) + table_span((size_t)width * 8);
    for (uint32_t c = threadIdx.x; c < width; c += blockDim.x) sL[c] = make_int2(CHP_EMPTY, CHP_EMPTY);
    __syncthreads();
    bool bad = false;
    auto f = [&](int32_t x, int32_t y) {
        uint32_t s;
        if (!accept<VALIDATE>(g, x, y, s)) {
            bad = true;
            return;
        }
        const int2 e = sL[s];
        if (y < e.x) atomicMin(&sL[s].x, y);
        if (~y < e.y) atomicMin(&sL[s].y, ~y);
    };
    stream_points<TMA>(xy, n, ring, stages, per_point4(f), f);
    pdl_wait();  // (a programmatic dependent of the DL init: only the flush touches DL)
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
// Slot word: bits 0-15 a = y - 1 (min), bits 16-31 b = 0xFFFF - a (min);
// empty = 0xFFFFFFFF.  Only for validated input with 1 <= y <= q <= 65536,
// so a = y - 1 always fits 16 bits and the point's own word is
//   pw = a | (0xFFFF - a) << 16 = 0xFFFF0000 - a * 0xFFFF.
// A point changes its slot iff vminu2(w, pw) != w (one VIMNMX.U16x2).  The
// hit path is branch-free with the shared base hoisted: the branchy form
// issued ~27 instructions per point (per-point S2UR of the shared window,
// three branches) and ran issue-bound (ncu C3: 79% issue-active).
template <bool TMA>
__global__ void __launch_bounds__(kThreads) k_reduce_smem16(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, int stages,
                                                            int* __restrict__ DL) {
    extern __shared__ uint4 smem4[];
    uint32_t* sW = reinterpret_cast<uint32_t*>(smem4);
    uint8_t* ring = reinterpret_cast<uint8_t*>(smem4) + table_span((size_t)width * 4);
    for (uint32_t c = threadIdx.x; c < width; c += blockDim.x) sW[c] = 0xFFFFFFFFu;
    __syncthreads();
    // Kernel constants pinned in ordinary registers: left to the compiler,
    // the shared window base (S2UR + ULEA) and the Geo words (LDCU) are
    // rematerialised for every point.
    const uint32_t tbase = pin((uint32_t)__cvta_generic_to_shared(smem4));
    const uint32_t base = pin(g.base), wcheck = pin(g.wcheck), qmax = pin(g.qmax), ybase = pin(g.ybase);
    uint32_t bad = 0;
    auto one = [&](int32_t x, int32_t y) {
        uint32_t s = slot_of(x, base);
        const uint32_t ym1 = (uint32_t)y - ybase;
        const bool ok = (s < wcheck) & (ym1 < qmax);
        bad |= !ok;
        s = ok ? s : 0u;
        const uint32_t pw = 0xFFFF0000u - ym1 * 0xFFFFu;
        uint32_t w = lds_u32(tbase + 4 * s);
        if (ok & (__vminu2(w, pw) != w)) {  // rare: the point moves an extreme
            for (;;) {
                const uint32_t nw = __vminu2(w, pw);
                if (nw == w) break;
                const uint32_t old = atomicCAS(sW + s, w, nw);
                if (old == w) break;
                w = old;
            }
        }
    };
    stream_points<TMA>(xy, n, ring, stages, per_point4(one), one, g.blocked != 0);
    // A programmatic dependent of the DL init: the stream above does not
    // touch DL, so only the flush waits for it.  Streaming the points before
    // the wait is valid because it can overlap only the immediate
    // predecessor, and no kernel that triggers its dependents early writes
    // points (they write DL, tables and snapshots; K3, the generators,
    // unpack and translate do not trigger early).
    pdl_wait();
    flag_error(bad != 0, DL, width);
    __syncthreads();
    int2* __restrict__ gL = reinterpret_cast<int2*>(DL);
    for (uint32_t c = threadIdx.x; c < width; c += blockDim.x) {
        const uint32_t w = sW[c];
        const uint32_t a = w & 0xFFFFu, b = w >> 16;
        if (a > 0xFFFFu - b) continue;  // lo > hi: empty
        const int32_t lo = (int32_t)(g.ybase + a);
        const int32_t nhi = ~(int32_t)(g.ybase + (0xFFFFu - b));
        const int2 cur = ld_cg2(gL + c);
        if (lo < cur.x) red_min(DL + 2ull * c, lo);
        if (nhi < cur.y) red_min(DL + 2ull * c + 1, nhi);
    }
}

// ------------------------------------------------------------ global
template <bool VALIDATE, bool TMA>
__global__ void __launch_bounds__(kThreads) k_reduce_global(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, int stages,
                                                            int* __restrict__ DL) {
    extern __shared__ uint4 smem4[];
    uint8_t* ring = reinterpret_cast<uint8_t*>(smem4);
    const int2* gL = reinterpret_cast<const int2*>(DL);
    bool bad = false;
    auto one = [&](int32_t x, int32_t y) {
        uint32_t s;
        if (!accept<VALIDATE>(g, x, y, s)) {
            bad = true;
            return;
        }
        const int2 e = ld_cg2(gL + s);
        if (y < e.x) red_min(DL + 2ull * s, y);
        if (~y < e.y) red_min(DL + 2ull * s + 1, ~y);
    };
    stream_points<TMA>(
        xy, n, ring, stages,
        [&](const int4& a, const int4& b) {
            int x[4], y[4];
            uint32_t s[4], miss = 0;
            unpack4(a, b, x, y);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (accept<VALIDATE>(g, x[k], y[k], s[k]))
                    miss |= 1u << k;
                else
                    bad = true;
            }
            settle_misses<true>(miss, s, y, DL);
        },
        one);
    flag_error(bad, DL, width);
}

// --------------------------------------------------- global, warp-aggregated
// north_star (a)'s form for large p or skewed columns: the lanes of a warp
// that hold the same slot elect one leader (__match_any_sync), which applies
// the group's min y and min ~y (__reduce_min_sync) with one read-compare-RED
// -- one L2 round trip per distinct slot per warp instead of per point.
// Invalid points share the match key 0xFFFFFFFF and are only flagged.
template <bool VALIDATE>
__global__ void __launch_bounds__(kThreads) k_reduce_global_agg(const int32_t* __restrict__ xy, uint64_t n, Geo g,
                                                                uint32_t width, int* __restrict__ DL) {
    const int2* gL = reinterpret_cast<const int2*>(DL);
    const uint32_t lane = threadIdx.x & 31;
    bool bad = false;
    // Every lane of the warp runs the same number of rounds (a lane past the
    // end contributes an invalid key that is not flagged).
    auto round = [&](bool live, int32_t x, int32_t y) {
        uint32_t s;
        const bool ok = live && accept<VALIDATE>(g, x, y, s);
        bad |= live && !ok;
        const uint32_t key = ok ? s : 0xFFFFFFFFu;
        const uint32_t grp = __match_any_sync(0xFFFFFFFFu, key);
        const int lo = (int)__reduce_min_sync(grp, (uint32_t)(y ^ INT_MIN)) ^ INT_MIN;  // signed min
        const int nhi = (int)__reduce_min_sync(grp, (uint32_t)(~y ^ INT_MIN)) ^ INT_MIN;
        if (ok && lane == (uint32_t)(__ffs(grp) - 1)) {
            const int2 e = ld_cg2(gL + s);
            if (lo < e.x) red_min(DL + 2ull * s, lo);
            if (nhi < e.y) red_min(DL + 2ull * s + 1, nhi);
        }
    };
    const Split sp = split_points(xy, n);
    const int4* __restrict__ v = reinterpret_cast<const int4*>(xy + 2 * sp.head);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
    for (uint64_t w = warp0; w < sp.nvec; w += stride) {
        const uint64_t i = w + lane;
        const bool live = i < sp.nvec;
        const int4 a = live ? ld_stream(v + i) : make_int4(0, 0, 0, 0);
        round(live, a.x, a.y);
        round(live, a.z, a.w);
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {  // the scalar head / tail points, by warp 0
        const bool h = sp.head && lane == 0, t = sp.tail && lane == 1;
        const int32_t* q = h ? xy : t ? xy + 2 * (n - 1) : xy;
        round(h || t, q[0], q[1]);
    }
    flag_error(bad, DL, width);
}

// ------------------------------------------------------------ filter
// Filter word per group of 2^gshift columns, two H-bit halves (H = 8 in a
// 16-bit word, or 16 in a 32-bit word): low half fa, high half span with
//   fa = ceil((max_lo - 1) / 2^ys),  fb = floor(min_hi / 2^ys) - 1,
//   span = min(fb - fa + 1, 2^H - 1)  (0 = never skip),
// and a point is skipped iff (u - fa) < span (unsigned) for u = (y - 1) >> ys,
// i.e. fa <= u <= fb, which implies max_lo <= y <= min_hi (DESIGN.md,
// "filter").  The table has ngroups + 1 words: word ngroups is the sink of
// invalid x (x clamps to slot `width`), and a partial last group is "never"
// too, so the clamp can only land on a never-skip word.
template <typename W>
struct FW {
    static constexpr uint32_t kHalf = sizeof(W) * 4;
    static constexpr uint32_t kMask = (1u << kHalf) - 1u;
    static constexpr W kNever = (W)0;  // span 0
};

template <typename W>
__device__ __forceinline__ uint32_t lds_w(uint32_t addr) {
    if (sizeof(W) == 2) {
        uint16_t v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
        return v;
    } else {
        return lds_u32(addr);
    }
}

// One thread per group, its columns read as 16-byte pairs with up to 8
// loads in flight (a warp-per-group form left half the lanes idle and ran
// one round trip per wave: 16 us per snapshot at p = 2^20).  Word
// `ngroups` (the sink) and a partial last group are "never".
// The snapshot word of group gi from DL (with the bucket base and shift);
// kLoads 16-byte loads in flight per thread.
template <typename W, int kLoads = 8>
__device__ __forceinline__ W filter_word(const int* __restrict__ DL, uint32_t width, uint32_t gshift,
                                         int32_t ybase, uint32_t ys, uint32_t gi, uint32_t ngroups) {
    const uint32_t c0 = gi << gshift;
    const uint32_t c1 = c0 + (1u << gshift);
    W word = FW<W>::kNever;
    if (gi < ngroups && c1 <= width) {
        int maxlo = INT32_MIN, minhi = INT32_MAX;
        bool empty = false;
        auto fold = [&](int lo, int nhi) {
            const int hi = ~nhi;
            empty |= lo > hi;
            maxlo = max(maxlo, lo);
            minhi = min(minhi, hi);
        };
        if (gshift >= 1 && !(reinterpret_cast<uintptr_t>(DL) & 15)) {  // 16-byte aligned pairs
            const int4* p4 = reinterpret_cast<const int4*>(DL) + (c0 >> 1);
            const uint32_t n4 = 1u << (gshift - 1);
            for (uint32_t i = 0; i < n4; i += kLoads) {
                int4 q[kLoads];
#pragma unroll
                for (int k = 0; k < kLoads; ++k)
                    if (i + k < n4) q[k] = __ldcg(p4 + i + k);
#pragma unroll
                for (int k = 0; k < kLoads; ++k)
                    if (i + k < n4) {
                        fold(q[k].x, q[k].y);
                        fold(q[k].z, q[k].w);
                    }
            }
        } else {
            const int2* p2 = reinterpret_cast<const int2*>(DL);
            for (uint32_t c = c0; c < c1; ++c) {
                const int2 e = ld_cg2(p2 + c);
                fold(e.x, e.y);
            }
        }
        if (!empty) {
            constexpr long long M = FW<W>::kMask;
            const long long q = 1ll << ys;
            const long long a = (long long)maxlo - ybase;
            const long long fa = a <= 0 ? 0 : (a + q - 1) / q;
            const long long b = (long long)minhi - ybase + 1;
            long long fb = b >= 0 ? b / q - 1 : -1;
            if (fb > M) fb = M;
            if (fa <= fb) {
                const long long span = (fb - fa + 1) < M ? (fb - fa + 1) : M;
                word = (W)((uint32_t)fa | ((uint32_t)span << FW<W>::kHalf));
            }
        }
    }
    return word;
}

// One thread per group, its columns read as 16-byte pairs with up to 8
// loads in flight (a warp-per-group form left half the lanes idle and ran
// one round trip per wave: 16 us per snapshot at p = 2^20).  Word
// `ngroups` (the sink) and a partial last group are "never".
template <typename W>
__global__ void __launch_bounds__(256) k_filter_build(const int* __restrict__ DL, uint32_t width, uint32_t gshift,
                                                      int32_t ybase, uint32_t ys, W* __restrict__ F,
                                                      uint32_t ngroups, const int2* __restrict__ qs) {
    pdl_trigger();  // the next phase may queue (its CTAs wait for this grid)
    pdl_wait();     // the previous phase's updates of DL
    const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi > ngroups) return;
    if (qs) {  // q unset: the speculative bucket range (k_quant_shift)
        const int2 v = __ldcg(qs);
        ybase = v.x;
        ys = (uint32_t)v.y;
    }
    F[gi] = filter_word<W>(DL, width, gshift, ybase, ys, gi, ngroups);
}

// F == nullptr starts from an all-"never skip" table (the warm-up pass:
// every point is settled in L2, building the first snapshot).  Validated
// input only (y in [1, q]); the host guarantees wcheck == width.
// The read-first register form runs 896 threads per CTA: its miss batches
// plus the load pipeline need more than 64 registers per thread (at 1024
// threads it spilled 32 B; C4: 768 656, 896 663, 1024 657 Gpts/s).
constexpr int kThreadsRF = 896;
template <typename W, bool READ_FIRST, bool TMA, bool SPEC>
__global__ void __launch_bounds__((READ_FIRST && !TMA) ? kThreadsRF : kThreads) k_reduce_filter(const int32_t* __restrict__ xy, uint64_t n,
                                                            Geo g, uint32_t width, uint32_t gshift, uint32_t ys,
                                                            const W* __restrict__ F, uint32_t ngroups, int stages,
                                                            int* __restrict__ DL, const int2* __restrict__ qs) {
    extern __shared__ uint4 sF4[];
    W* sF = reinterpret_cast<W*>(sF4);
    const uint32_t nwords = ngroups + 1;
    uint8_t* ring = reinterpret_cast<uint8_t*>(sF4) + table_span((size_t)nwords * sizeof(W));
    // Launched as a programmatic dependent of the snapshot build (or of the
    // DL init): the next build may queue at once, and this grid waits for
    // its predecessor's table (and DL) before reading them.
    pdl_trigger();
    pdl_wait();
    {
        const uint32_t per4 = 16 / sizeof(W);
        const uint32_t n4 = nwords / per4;
        if (F) {
            const uint4* F4 = reinterpret_cast<const uint4*>(F);
            for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) sF4[i] = __ldcg(F4 + i);
            for (uint32_t i = n4 * per4 + threadIdx.x; i < nwords; i += blockDim.x) sF[i] = F[i];
        } else {
            for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) sF[i] = FW<W>::kNever;
        }
    }
    // Bucket base: the valid range's (q known), or the speculative range's
    // (q unset: k_quant_shift); a y below it wraps past every bucket and
    // misses, one above it has u > every fb and misses.
    uint32_t qb = g.ybase;
    if (SPEC) {
        const int2 v = __ldcg(qs);
        qb = (uint32_t)v.x;
        ys = (uint32_t)v.y;
    }
    __syncthreads();
    constexpr uint32_t H = FW<W>::kHalf, HM = FW<W>::kMask;
    const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(sF4);
    uint32_t bad = 0;
    // Branch-free hit test: true when the point must be settled.  An invalid
    // x reads a never-skip word; an invalid y has u > fb (or wraps), so it
    // misses as well and is caught in the miss path.
    auto test = [&](int32_t x, int32_t y, uint32_t& s, uint32_t& w) -> bool {
        s = min(slot_of(x, g.base), width);
        w = lds_w<W>(tbase + (s >> gshift) * (uint32_t)sizeof(W));
        return (((uint32_t)y - qb) >> ys) - (w & HM) >= (w >> H);
    };
    auto valid = [&](uint32_t s, int32_t y) {
        const bool ok = (s < g.wcheck) & ((uint32_t)y - g.ybase < g.qmax);
        bad |= !ok;
        return ok;
    };
    // RED-only misses are one-sided where the word allows: u <= fb means
    // y <= min_hi of the group, so only lo can move; u >= fa means
    // y >= max_lo, so only hi can move.
    auto settle_red = [&](uint32_t s, int32_t y, uint32_t w) {
        if (!valid(s, y)) return;
        const uint32_t fa = w & HM, span = w >> H;
        if (SPEC && y < (int32_t)qb) {  // below the speculative range: below max_lo's bucket, <= min_hi
            red_min(DL + 2ull * s, y);
            if (span == 0) red_min(DL + 2ull * s + 1, ~y);
            return;
        }
        const uint32_t u = ((uint32_t)y - qb) >> ys;
        if (span == 0 || u > fa) red_min(DL + 2ull * s + 1, ~y);  // not known below min_hi
        if (span == 0 || u < fa) red_min(DL + 2ull * s, y);       // not known above max_lo
    };
    auto one = [&](int32_t x, int32_t y) {
        uint32_t s, w;
        if (!test(x, y, s, w)) return;
        if (READ_FIRST) {
            if (!valid(s, y)) return;
            uint32_t ss[1] = {s};
            int yy[1] = {y};
            settle_misses<true>(1u, ss, yy, DL);
        } else {
            settle_red(s, y, w);
        }
    };
    if (READ_FIRST) {
        // Four tests, then the misses' L2 reads all in flight together.
        stream_points<TMA>(
            xy, n, ring, stages,
            [&](const int4& a, const int4& b) {
                const int y[4] = {a.y, a.w, b.y, b.w};
                uint32_t s[4], w, miss = 0;  // (the words are not needed here: one scratch)
                miss |= (uint32_t)test(a.x, a.y, s[0], w);
                miss |= (uint32_t)test(a.z, a.w, s[1], w) << 1;
                miss |= (uint32_t)test(b.x, b.y, s[2], w) << 2;
                miss |= (uint32_t)test(b.z, b.w, s[3], w) << 3;
                if (miss) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (((miss >> k) & 1) && !valid(s[k], y[k])) miss &= ~(1u << k);
                    settle_misses<true>(miss, s, y, DL);
                }
            },
            one, g.blocked != 0);
    } else {
        stream_points<TMA>(xy, n, ring, stages, per_point4(one), one, g.blocked != 0);
    }
    flag_error(bad != 0, DL, width);
}

// ------------------------------------------------------------ sampled
// Per-column filter built from a sample, exact by construction (mid-size p,
// DESIGN.md "sampled filter").  Buckets u = umulhi(y - base, m) (Quant) chosen so
// that u <= 254.
//  1. k_sample_learn: each CTA folds its share of a sample (a prefix of the
//     input) into a private table of (ua, ub) = (min, max) bucket per column
//     with plain, racy shared-memory stores -- no atomics, no global traffic.
//     Every stored endpoint is the bucket of an actual sample point (a lost
//     race only narrows the interval).  Tables go to scratch.
//  2. k_sample_merge: per column ua = min, ub = max over the CTA tables; the
//     main-pass word is the STRICT interior: lo = ua + 1, span = ub - lo
//     (>= 0), skip iff (u - lo) < span (unsigned) i.e. ua < u < ub.
//  3. k_reduce_sampled: one pass over ALL points.  A skipped point lies
//     strictly between two sample points of its column, which are never
//     skipped themselves (they sit in the boundary buckets) and so reach L:
//     the skipped point cannot be an extreme.  A miss with span > 0 lies at
//     or beyond one boundary bucket, so only that side can move: one RED,
//     then the word widens to the point's bucket.
// Tables are dumped as (ua, 255 - ub) so the merge is one byte-wise min.
// With init_dl the kernel also initialises DL (the main pass runs after it in
// stream order), saving the separate k_dl_init launch.
// Quantisation of y into the table's buckets: u = umulhi(y - base, m), in
// [0, 254] over the range the table covers.  With q known the range is the
// valid range (base = ybase); with q unset (validation only y >= ybase) it is
// speculative, [min, max] of the valid y in a 2^18-point prefix (k_yrange, one partial
// per CTA, reduced by every consumer CTA): a point outside it is still exact,
// it folds into the edge bucket and always misses the main-pass test (below
// the base its offset wraps past every bucket), and settle moves the side it
// lies on.
struct Quant {
    int32_t base;
    uint32_t m;
};

__host__ __device__ inline uint32_t quant_mult(uint64_t count) {
    const uint64_t m = ((uint64_t)255 << 32) / (count ? count : 1);
    return m > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)m;
}

// One round trip: a 2^18-point prefix over 148 x 1024 threads.
__global__ void __launch_bounds__(1024) k_yrange(const int32_t* __restrict__ xy, uint64_t n, Geo g,
                                                 int2* __restrict__ part) {
    __shared__ int2 red[32];
    int lo = INT_MAX, hi = INT_MIN;
    auto f = [&](int32_t x, int32_t y) {
        uint32_t s;
        if (accept<true>(g, x, y, s)) {
            lo = min(lo, y);
            hi = max(hi, y);
        }
    };
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const int2 p = reinterpret_cast<const int2*>(xy)[i];
        f(p.x, p.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_int2(lo, hi);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            lo = min(lo, red[k].x);
            hi = max(hi, red[k].y);
        }
        part[blockIdx.x] = make_int2(lo, hi);
    }
}

// Every CTA derives the same Quant from the k_yrange partials (warp 0
// reduces them; the result is broadcast through shared memory).
__device__ __forceinline__ Quant resolve_quant(Quant qz, const int2* __restrict__ part, uint32_t np, const Geo& g) {
    if (!part) return qz;
    __shared__ Quant s_q;
    if (threadIdx.x < 32) {
        int lo = INT_MAX, hi = INT_MIN;
        for (uint32_t i = threadIdx.x; i < np; i += 32) {
            const int2 v = __ldcg(part + i);
            lo = min(lo, v.x);
            hi = max(hi, v.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (threadIdx.x == 0) {
            Quant r;
            if (lo > hi) {  // no valid y in the prefix: the whole valid range
                r.base = (int32_t)g.ybase;
                r.m = quant_mult(g.qmax);
            } else {
                r.base = lo;
                r.m = quant_mult((uint64_t)((int64_t)hi - lo + 1));
            }
            s_q = r;
        }
    }
    __syncthreads();
    return s_q;
}

// The group filter's form of the same (one CTA): {base, ys} with the
// speculative range >> ys <= kmask, written to qs for every later kernel.
__global__ void k_quant_shift(const int2* __restrict__ part, uint32_t np, Geo g, uint32_t kmask,
                              int2* __restrict__ qs) {
    int lo = INT_MAX, hi = INT_MIN;
    for (uint32_t i = threadIdx.x; i < np; i += 32) {
        const int2 v = part[i];
        lo = min(lo, v.x);
        hi = max(hi, v.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (threadIdx.x == 0) {
        uint64_t ext;
        if (lo > hi) {
            lo = (int)g.ybase;
            ext = (uint64_t)g.qmax - 1;
        } else {
            ext = (uint64_t)((int64_t)hi - lo);
        }
        uint32_t ys = 0;
        while ((ext >> ys) > kmask) ++ys;
        *qs = make_int2(lo, (int)ys);
    }
}

// Phase helpers shared by the three-launch pipeline and the fused kernel.
__device__ __forceinline__ void sample_init(uint4* smem4, uint32_t wpad, int* __restrict__ DL, uint32_t width,
                                            int init_dl) {
    for (uint32_t c = threadIdx.x; smem4 && c < wpad / 8; c += blockDim.x)  // ua = 255 > ub = 0: empty
        smem4[c] = make_uint4(0x00FF00FFu, 0x00FF00FFu, 0x00FF00FFu, 0x00FF00FFu);
    if (init_dl) {
        const uint64_t words = 2ull * width;
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
             i += (uint64_t)gridDim.x * blockDim.x)
            DL[i] = CHP_EMPTY;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            DL[words] = 0;
            DL[words + 1] = 0;
        }
    }
}

// Fold this CTA's share of the sample into T.  No validation here: an
// invalid x lands in the sink slot `width` (never merged), an invalid y can
// only garble its own column's word, and the main pass, which sees every
// point again, fails the call.
//
// The sample is n * f256 / 256 points: by default the head of every CTA's
// main-pass slice (for_each_group_pp's [vb, ve)); `prefix` (and the TMA form)
// take the first n * f256 / 256 points instead.  The heads spread the sample
// over the whole input (an input sorted by x or y still yields a table for
// every part of it); on C2 the two measure the same.
template <bool TMA, bool SPEC>
__device__ __forceinline__ void sample_fold(const int32_t* __restrict__ xy, uint64_t n, uint32_t f256, bool prefix,
                                            const Geo& g, uint32_t width, Quant qz, uint16_t* T, uint8_t* ring,
                                            int stages) {
    auto f = [&](int32_t x, int32_t y) {
        const uint32_t s = min(slot_of(x, g.base), width);
        // Outside the quantised range: the edge bucket (0 or 254).
        // (q known: every valid y is in range; an invalid one may garble its
        // own column's word, and the main pass fails the call.)
        const uint32_t uq = __umulhi((uint32_t)y - (uint32_t)qz.base, qz.m);
        const uint32_t u = SPEC ? (y < qz.base ? 0u : min(uq, 254u)) : uq;
        const uint32_t w = T[s];
        const uint32_t nw = min(w & 0xFFu, u) | (max(w >> 8, u) << 8);
        if (nw != w) T[s] = (uint16_t)nw;
    };
    if (TMA) {
        const uint64_t ns = n * f256 >> 8;
        stream_points<true>(xy, ns > 2 ? ns : (n < 2 ? n : 2), ring, stages, per_point4(f), f);
        return;
    }
    // Each thread sees only ~80 sample points, so the pass is bound by
    // round trips, not bandwidth: a batch of vectors per thread is issued at
    // once (3 round trips instead of 10 for the C2 sample).
    const Split sp = split_points(xy, n);
    const int4* __restrict__ v = reinterpret_cast<const int4*>(xy + 2 * sp.head);
    uint64_t stride, i, end;
    if (prefix) {
        stride = (uint64_t)gridDim.x * blockDim.x;
        i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        end = sp.nvec * f256 >> 8;
    } else {
        const uint64_t vb = sp.nvec * blockIdx.x / gridDim.x, ve = sp.nvec * (blockIdx.x + 1) / gridDim.x;
        stride = blockDim.x;
        i = vb + threadIdx.x;
        end = vb + ((ve - vb) * f256 >> 8);
    }
    constexpr int kB = 16;  // loads issued per batch (C2: 8 575.6, 12 577.3, 16 578.5 Gpts/s)
    for (; i + (kB - 1) * stride < end; i += kB * stride) {
        int4 q[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) q[j] = ld_stream(v + i + j * stride);
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            f(q[j].x, q[j].y);
            f(q[j].z, q[j].w);
        }
    }
    for (; i < end; i += stride) {
        const int4 a = ld_stream(v + i);
        f(a.x, a.y);
        f(a.z, a.w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (sp.head) f(xy[0], xy[1]);
        if (sp.tail) f(xy[2 * (n - 1)], xy[2 * (n - 1) + 1]);
    }
}

// This CTA's table to scratch as (ua, 255 - ub), so the merge is one
// byte-wise min.
__device__ __forceinline__ void sample_dump(const uint4* smem4, uint16_t* __restrict__ scratch, uint32_t wpad) {
    uint4* dst = reinterpret_cast<uint4*>(scratch + (size_t)blockIdx.x * wpad);
    for (uint32_t i = threadIdx.x; i < wpad / 8; i += blockDim.x) {
        uint4 q = smem4[i];
        q.x ^= 0xFF00FF00u;
        q.y ^= 0xFF00FF00u;
        q.z ^= 0xFF00FF00u;
        q.w ^= 0xFF00FF00u;
        dst[i] = q;
    }
}

__device__ __forceinline__ void vmin4x4(uint4& m, const uint4& q) {
    m.x = __vminu4(m.x, q.x);
    m.y = __vminu4(m.y, q.y);
    m.z = __vminu4(m.z, q.z);
    m.w = __vminu4(m.w, q.w);
}

// Merged (ua, 255 - ub) bytes of 8 columns -> 8 main-pass words: the strict
// interior lo = ua + 1, span = ub - lo; columns >= width (incl. the sink) and
// empty columns get lo = 255, span = 0 (never skip).
__device__ __forceinline__ uint4 interior_words(const uint4& m, uint32_t chunk, uint32_t width) {
    const uint32_t words[4] = {m.x, m.y, m.z, m.w};
    uint32_t out[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t o = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t c = chunk * 8 + k * 2 + h;
            const uint32_t w16 = (words[k] >> (16 * h)) & 0xFFFFu;
            const uint32_t ua = w16 & 0xFFu, ub = 255u - (w16 >> 8);
            uint32_t word = 0x00FF;
            if (c < width && ua <= ub) {
                const uint32_t lo = ua + 1;  // <= 255 because buckets stop at 254
                word = lo | ((ub > lo ? ub - lo : 0) << 8);
            }
            o |= word << (16 * h);
        }
        out[k] = o;
    }
    return make_uint4(out[0], out[1], out[2], out[3]);
}

template <bool TMA, bool SPEC>
__global__ void __launch_bounds__(kThreads) k_sample_learn(const int32_t* __restrict__ xy, uint64_t n, Geo g,
                                                           uint32_t width, uint32_t wpad, Quant qz,
                                                           const int2* __restrict__ qpart, uint32_t nqpart,
                                                           uint16_t* __restrict__ scratch, int* __restrict__ DL,
                                                           int init_dl, int stages, uint32_t f256, int prefix) {
    extern __shared__ uint4 smem4[];
    uint8_t* ring = reinterpret_cast<uint8_t*>(smem4) + table_span((size_t)wpad * 2);
    pdl_trigger();  // the merge may queue (it cannot co-reside; it waits)
    if (SPEC) qz = resolve_quant(qz, qpart, nqpart, g);
    sample_init(smem4, wpad, DL, width, init_dl);
    __syncthreads();
    sample_fold<TMA, SPEC>(xy, n, f256, prefix != 0, g, width, qz, reinterpret_cast<uint16_t*>(smem4), ring, stages);
    __syncthreads();
    sample_dump(smem4, scratch, wpad);
}

// Byte-wise min over the CTA tables: thread (x, y) folds tables y, y+16, ...
// for 8 columns (one uint4) with all its loads in flight at once (a single
// round trip for <= 160 tables), then the 16 partials meet in shared memory.
constexpr int kMergeCols = 16;    // uint4 chunks per block (x)
constexpr int kMergeSlices = 16;  // table slices per block (y)
constexpr int kMergeBatch = 10;   // loads in flight per thread

__global__ void __launch_bounds__(kMergeCols * kMergeSlices) k_sample_merge(const uint16_t* __restrict__ scratch,
                                                                           uint32_t ntables, uint32_t width,
                                                                           uint32_t wpad, uint16_t* __restrict__ F) {
    __shared__ uint4 part[kMergeSlices][kMergeCols];
    pdl_trigger();
    pdl_wait();  // the sample tables
    const uint32_t chunk = blockIdx.x * kMergeCols + threadIdx.x;
    const uint32_t nchunks = wpad / 8;
    const uint4 ones = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    uint4 m = ones;
    if (chunk < nchunks) {
        const uint4* src = reinterpret_cast<const uint4*>(scratch) + chunk;
        for (uint32_t t0 = threadIdx.y; t0 < ntables; t0 += kMergeSlices * kMergeBatch) {
            uint4 q[kMergeBatch];
#pragma unroll
            for (int k = 0; k < kMergeBatch; ++k) {
                const uint32_t t = t0 + k * kMergeSlices;
                q[k] = t < ntables ? __ldcs(src + (size_t)t * nchunks) : ones;
            }
#pragma unroll
            for (int k = 0; k < kMergeBatch; ++k) vmin4x4(m, q[k]);
        }
    }
    part[threadIdx.y][threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.y != 0 || chunk >= nchunks) return;
    for (int k = 1; k < kMergeSlices; ++k) vmin4x4(m, part[k][threadIdx.x]);
    reinterpret_cast<uint4*>(F)[chunk] = interior_words(m, chunk, width);
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((uint16_t)v) : "memory");
}

// The main pass over all n points against the strict-interior table at
// shared address tbase (>= width + 1 words; word `width` never skips).
template <bool TMA, bool SPEC>
__device__ __forceinline__ void sampled_pass(const int32_t* __restrict__ xy, uint64_t n, const Geo& g,
                                             uint32_t width, Quant qz, uint32_t tbase, uint8_t* ring,
                                             int stages, int* __restrict__ DL) {
    uint32_t bad = 0;
    // Rare path: a point outside the strict interior of its column.  Inlined
    // (an out-of-line __noinline__ version measured 411 vs 491 Gpts/s).
    // Validation lives here too: an invalid point always reaches it (below).
    auto settle = [&](uint32_t s, int32_t y) {
        const uint32_t ym1 = (uint32_t)y - g.ybase;
        if (s >= g.wcheck || ym1 >= g.qmax) {
            bad = 1;
            return;
        }
        CHP_CHECK(s < width);
        const uint32_t a = tbase + 2 * s;
        const uint32_t w = lds_u16(a);
        const uint32_t lo = w & 0xFFu, span = w >> 8;
        if (span == 0) {  // nothing known: both sides may move
            red_min(DL + 2ull * s, y);
            red_min(DL + 2ull * s + 1, ~y);
            return;
        }
        // SPEC (q unset): below the quantised range counts as bucket -1,
        // above it as bucket 255 (past every stored bucket).  Otherwise every
        // valid y is in range.
        const bool below = SPEC && y < qz.base;
        const uint32_t uq = __umulhi((uint32_t)y - (uint32_t)qz.base, qz.m);
        const uint32_t u = SPEC ? (below ? 0u : min(uq, 255u)) : uq;
        if (below || u < lo) {  // at/below the lower boundary bucket: only lo moves
            red_min(DL + 2ull * s, y);
            const uint32_t nlo = below ? 0u : u + 1;
            if (nlo < lo) sts_u16(a, nlo | ((lo + span - nlo) << 8));
        } else if (u >= lo + span) {  // at/above the upper boundary bucket: only hi moves
            red_min(DL + 2ull * s + 1, ~y);
            if (u > lo + span) sts_u16(a, lo | ((u - lo) << 8));
        }
    };
    // Hit test of one point, branch-free: true when it must be settled.  An
    // invalid x clamps to slot `width`, whose word (span 0) never skips (the
    // host guarantees wcheck == width and a table of at least width + 1
    // slots); an invalid y has a bucket >= every ub of a strict
    // interior (or wraps), so it misses too.  Validation thus costs one
    // VIADDMNMX per point instead of two compares, a select and a flag.
    auto test = [&](int32_t x, int32_t y, uint32_t& s) -> bool {
        s = min(slot_of(x, g.base), width);
        const uint32_t w = lds_u16(tbase + 2 * s);
        const uint32_t lo = w & 0xFFu, span = w >> 8;
        return __umulhi((uint32_t)y - (uint32_t)qz.base, qz.m) - lo >= span;  // not strictly inside
    };
    auto one = [&](int32_t x, int32_t y) {
        uint32_t s;
        if (test(x, y, s)) settle(s, y);
    };
    // Four points: branch-free tests, then the (rare) misses.
    auto g4 = [&](const int4& a, const int4& b) {
        const int y[4] = {a.y, a.w, b.y, b.w};
        uint32_t s[4], miss = 0;
        miss |= (uint32_t)test(a.x, a.y, s[0]);
        miss |= (uint32_t)test(a.z, a.w, s[1]) << 1;
        miss |= (uint32_t)test(b.x, b.y, s[2]) << 2;
        miss |= (uint32_t)test(b.z, b.w, s[3]) << 3;
        if (miss) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if ((miss >> k) & 1) settle(s[k], y[k]);
        }
    };
    // Register path: per point (a batched form spilled at 64 registers and
    // measured 462 vs 482 Gpts/s on C2).
    auto g8 = [&](const int4& a, const int4& b, const int4& c, const int4& d) {
        one(a.x, a.y); one(a.z, a.w);
        one(b.x, b.y); one(b.z, b.w);
        one(c.x, c.y); one(c.z, c.w);
        one(d.x, d.y); one(d.z, d.w);
    };
    if (TMA)
        stream_points<true>(xy, n, ring, stages, g4, one);
    else
        for_each_group_pp(xy, n, g8, one);
    flag_error(bad != 0, DL, width);
}

template <bool TMA, bool SPEC>
__global__ void __launch_bounds__(kThreads) k_reduce_sampled(const int32_t* __restrict__ xy, uint64_t n, Geo g,
                                                             uint32_t width, uint32_t wpad, Quant qz,
                                                             const int2* __restrict__ qpart, uint32_t nqpart,
                                                             const uint16_t* __restrict__ F, int stages,
                                                             int* __restrict__ DL) {
    extern __shared__ uint4 smem4[];
    uint8_t* ring = reinterpret_cast<uint8_t*>(smem4) + table_span((size_t)wpad * 2);
    pdl_trigger();
    pdl_wait();  // the merged table (and DL, initialised by the sample pass)
    phase_mark(6);
    if (SPEC) qz = resolve_quant(qz, qpart, nqpart, g);
    {
        const uint4* F4 = reinterpret_cast<const uint4*>(F);
        for (uint32_t i = threadIdx.x; i < wpad / 8; i += blockDim.x) smem4[i] = __ldcg(F4 + i);
    }
    __syncthreads();
    sampled_pass<TMA, SPEC>(xy, n, g, width, qz, (uint32_t)__cvta_generic_to_shared(smem4), ring, stages, DL);
    if (CHP_PHASE_TIMING) {
        __syncthreads();
        phase_mark(7);
    }
}

// ------------------------------------------------------- sampled, fused
// The sampled pipeline as ONE cooperative kernel (all CTAs co-resident, one
// per SM): sample pass -> grid barrier -> merge, each CTA owning 1/grid of
// the columns -> grid barrier -> every CTA loads the merged table -> main
// pass.  Saves two launch boundaries (ramp-down/ramp-up) and spreads the
// merge over every SM.
// (GridBar / grid_barrier: chp_internal.cuh, shared with the cooperative K4.)
constexpr size_t kFusedMergeSmem = 16 * 64 * sizeof(uint4);  // phase B partials


// Out of line so phases A-C do not constrain the main pass's registers.
__device__ __noinline__ void sampled_main_pass(const int32_t* __restrict__ xy, uint64_t n, Geo g, uint32_t width,
                                               Quant qz, uint32_t tbase, int* __restrict__ DL) {
    sampled_pass<false, true>(xy, n, g, width, qz, tbase, nullptr, 0, DL);
}

template <bool SPEC>
__global__ void __launch_bounds__(kThreads) k_sampled_fused(const int32_t* __restrict__ xy, uint64_t n, uint32_t f256,
                                                            int prefix,
                                                            Geo g, uint32_t width, uint32_t wpad, Quant qz,
                                                            const int2* __restrict__ qpart, uint32_t nqpart,
                                                            uint16_t* __restrict__ scratch, uint16_t* __restrict__ F,
                                                            int* __restrict__ DL, int init_dl, GridBar* bar,
                                                            int merge_only) {
    extern __shared__ uint4 smem4[];
    const uint32_t nchunks = wpad / 8;
    if (merge_only) pdl_trigger();  // the main pass (a dependent launch) may queue
    phase_mark(0);
    if (SPEC) qz = resolve_quant(qz, qpart, nqpart, g);
    // ---- A: sample pass, then DL init.  Launched as a programmatic
    // dependent (when the runtime allows it with a cooperative launch), the
    // fold of the points runs before waiting for the predecessor (the
    // previous call's K3, which reads DL); only the DL init waits.
    sample_init(smem4, wpad, DL, width, 0);
    __syncthreads();
    phase_mark(1);
    sample_fold<false, SPEC>(xy, n, f256, prefix != 0, g, width, qz, reinterpret_cast<uint16_t*>(smem4), nullptr, 0);
    pdl_wait();
    if (init_dl) sample_init(nullptr, 0, DL, width, 1);
    __syncthreads();
    phase_mark(2);
    sample_dump(smem4, scratch, wpad);
    phase_mark(3);
    grid_barrier(bar);
    if (merge_only) grid_barrier_done(bar);
    phase_mark(4);
    // ---- B: merge; this CTA owns chunks [c0, c1), 64 chunks x 16 slices
    {
        const uint32_t per = (nchunks + gridDim.x - 1) / gridDim.x;
        const uint32_t c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
        uint4* part = smem4;  // [16][64] uint4, the table is reloaded in C
        const uint4 ones = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        for (uint32_t base = c0; base < c1; base += 64) {
            const uint32_t cl = threadIdx.x & 63, slice = threadIdx.x >> 6;
            const uint32_t chunk = base + cl;
            uint4 m = ones;
            if (chunk < c1) {
                const uint4* src = reinterpret_cast<const uint4*>(scratch) + chunk;
                for (uint32_t t0 = slice; t0 < gridDim.x; t0 += 16 * kMergeBatch) {
                    uint4 q[kMergeBatch];
#pragma unroll
                    for (int k = 0; k < kMergeBatch; ++k) {
                        const uint32_t t = t0 + k * 16;
                        q[k] = t < gridDim.x ? __ldcg(src + (size_t)t * nchunks) : ones;
                    }
#pragma unroll
                    for (int k = 0; k < kMergeBatch; ++k) vmin4x4(m, q[k]);
                }
            }
            part[slice * 64 + cl] = m;
            __syncthreads();
            if (slice == 0 && chunk < c1) {
                for (int k = 1; k < 16; ++k) vmin4x4(m, part[k * 64 + cl]);
                reinterpret_cast<uint4*>(F)[chunk] = interior_words(m, chunk, width);
            }
            __syncthreads();
        }
    }
    phase_mark(5);
    if (merge_only) return;  // the main pass is a separate (dependent) launch
    grid_barrier(bar);
    grid_barrier_done(bar);
    // ---- C: every CTA loads the merged table
    {
        const uint4* F4 = reinterpret_cast<const uint4*>(F);
        for (uint32_t i = threadIdx.x; i < nchunks; i += blockDim.x) smem4[i] = __ldcg(F4 + i);
    }
    __syncthreads();
    // ---- D: main pass
    sampled_main_pass(xy, n, g, width, qz, (uint32_t)__cvta_generic_to_shared(smem4), DL);
}


// ------------------------------------------------------------ filter8
// Per-column learning filter for mid-size p (one 16-bit word per column:
// bits 0-7 qa = ceil((lo-1) / 2^ys), bits 8-15 qb = floor(hi / 2^ys) - 1,
// "never skip" = 0x00FF).  A point with u = (y-1) >> ys in [qa, qb] has
// lo <= y <= hi for the column's current extremes and is skipped.  A miss
// reads the column from L2 (ld.cg), REDs what it improves and writes the
// tightened word back to shared memory, so each CTA's filter converges to
// the global L as the pass proceeds.
__device__ __forceinline__ uint16_t quant8(int lo, int hi, uint32_t ys) {
    if (lo > hi || lo < 1) return 0x00FF;
    const uint32_t a = ((uint32_t)(lo - 1) + ((1u << ys) - 1)) >> ys;
    const int b = (int)((uint32_t)hi >> ys) - 1;
    if (b < 0 || a > 255u || (int)a > b) return 0x00FF;
    return (uint16_t)(a | ((uint32_t)min(b, 255) << 8));
}

__global__ void k_filter8_build(const int* __restrict__ DL, uint32_t width, uint32_t ys, uint16_t* __restrict__ F) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= width) return;
    const int2 e = ld_cg2(reinterpret_cast<const int2*>(DL) + c);
    F[c] = quant8(e.x, ~e.y, ys);
}

template <bool TMA>
__global__ void __launch_bounds__(kThreads) k_reduce_filter8(const int32_t* __restrict__ xy, uint64_t n, Geo g,
                                                             uint32_t width, uint32_t ys,
                                                             const uint16_t* __restrict__ F, int stages,
                                                             int* __restrict__ DL) {
    extern __shared__ uint4 smem4[];
    uint16_t* sF8 = reinterpret_cast<uint16_t*>(smem4);
    uint8_t* ring = reinterpret_cast<uint8_t*>(smem4) + table_span((size_t)((width + 7) & ~7u) * 2);
    {
        const uint4* F4 = reinterpret_cast<const uint4*>(F);
        uint4* s4 = reinterpret_cast<uint4*>(sF8);
        const uint32_t n4 = width / 8;
        for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) s4[i] = __ldcg(F4 + i);
        for (uint32_t i = n4 * 8 + threadIdx.x; i < width; i += blockDim.x) sF8[i] = F[i];
    }
    __syncthreads();
    // A word (qa <= qb) asserts lo <= qa*2^ys + 1 and hi >= (qb+1)*2^ys.  A
    // point below that range can only lower lo, one above it only raise hi:
    // one RED, then the word widens to include y (still true afterwards).
    bool bad = false;
    auto one = [&](int32_t x, int32_t y) {
        uint32_t s;
        if (!accept<true>(g, x, y, s)) {
            bad = true;
            return;
        }
        const uint32_t f = sF8[s];
        const uint32_t qa = f & 0xFFu, qb = f >> 8;
        const uint32_t u = ((uint32_t)y - g.ybase) >> ys;
        if (u >= qa && u <= qb) return;
        if (qa > qb) {  // nothing known: both extremes may move
            red_min(DL + 2ull * s, y);
            red_min(DL + 2ull * s + 1, ~y);
            return;
        }
        if (u < qa) {
            red_min(DL + 2ull * s, y);
            sF8[s] = (uint16_t)((((uint32_t)(y - 1) + ((1u << ys) - 1)) >> ys) | (qb << 8));
        } else {
            red_min(DL + 2ull * s + 1, ~y);
            sF8[s] = (uint16_t)(qa | (min(((uint32_t)y >> ys) - 1u, 255u) << 8));
        }
    };
    stream_points<TMA>(xy, n, ring, stages, per_point4(one), one);
    flag_error(bad, DL, width);
}

// Launch plan of one K1 kernel: table bytes in shared memory plus, when TMA
// staging is on, a ring of as many 32 KB stages as fit (2..kMaxStages).
// Per-variant defaults come from measurement ("K1 tuning"):
// smem32 streams through the ring (its 128 KB table leaves one CTA/SM and
// the ring restores the bytes in flight: C3 697 vs 673 Gpts/s); smem16 and
// the filters stream through registers (C3 711 vs 568, C5 886 vs 702,
// C2 417 vs 406).  CHP_REDUCE_TMA / CHP_REDUCE_NO_TMA override.
constexpr int kMaxStages = 4;  // tools/micro_tma.cu: 4 x 32 KB beats 2 and 6

struct Plan {
    bool tma;
    int stages;
    size_t smem;
};

Plan plan_for(const chp_ctx* ctx, size_t table_bytes, uint32_t flags, bool tma_default) {
    Plan p{false, 0, table_span(table_bytes)};
    const bool want = (flags & CHP_REDUCE_TMA) ? true : (flags & CHP_REDUCE_NO_TMA) ? false : tma_default;
    if (!want) return p;
    const size_t limit = (size_t)ctx->smem_optin - 1024;
    if (p.smem >= limit) return p;
    int st = (int)((limit - p.smem) / chpstream::ring_bytes(1));
    if (st > kMaxStages) st = kMaxStages;
    if (st < 2) return p;
    p.tma = true;
    p.smem += chpstream::ring_bytes(st);
    p.stages = st;
    return p;
}

// Grid size for a kThreads kernel with `smem` dynamic shared memory, setting
// the kernel's smem attribute first.  Cached per context: the attribute call
// and the occupancy query cost microseconds of host time per launch, which
// the bench's launch rate (4 launches per 0.17 ms step) notices.
int kernel_blocks(chp_ctx* ctx, const void* fn, size_t smem, int cap_per_sm, int* blocks) {
    auto it = ctx->kcache.find(fn);
    int per_sm;
    if (it != ctx->kcache.end() && it->second.first == smem) {
        per_sm = it->second.second;
    } else {
        CHP_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        per_sm = 0;
        CHP_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
        ctx->kcache[fn] = {smem, per_sm};
    }
    if (per_sm < 1) per_sm = 1;
    if (per_sm > cap_per_sm) per_sm = cap_per_sm;
    *blocks = per_sm * ctx->sm_count;
    return CHP_OK;
}

// Launches kernel template K<..., TMA> with the plan's dynamic shared memory.
#define CHP_LAUNCH_PLANNED(ctx, plan, KTMA, KREG, ...)                                                   \
    do {                                                                                                 \
        auto fn_ = (plan).tma ? (KTMA) : (KREG);                                                         \
        int blocks_ = 0;                                                                                 \
        if (int rc_ = kernel_blocks((ctx), (const void*)fn_, (plan).smem, 2, &blocks_)) return rc_;     \
        fn_<<<blocks_, kThreads, (plan).smem, (ctx)->stream>>>(__VA_ARGS__);                            \
        CHP_LAUNCHED(ctx);                                                                               \
    } while (0)

// As CHP_LAUNCH_PLANNED, launched as a programmatic dependent of the
// previous kernel on the stream (the kernel calls pdl_wait()).
#define CHP_LAUNCH_PLANNED_PDL(ctx, plan, KTMA, KREG, ...)                                               \
    do {                                                                                                 \
        auto fn_ = (plan).tma ? (KTMA) : (KREG);                                                         \
        int blocks_ = 0;                                                                                 \
        if (int rc_ = kernel_blocks((ctx), (const void*)fn_, (plan).smem, 2, &blocks_)) return rc_;     \
        CHP_CUDA((ctx), launch_pdl(fn_, dim3(blocks_), dim3(kThreads), (plan).smem, (ctx)->stream, __VA_ARGS__)); \
        CHP_LAUNCHED(ctx);                                                                               \
    } while (0)

// Column-group snapshot filter in phases of doubling length (below), each
// against a fresh snapshot of DL.  The table (W = 16-bit
// words with 8-bit halves, or 32-bit words with 16-bit halves) is sized to
// `fbudget` bytes; the rest of shared memory holds the TMA ring.
template <typename W, bool SPEC>
int run_group_filter(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, const Geo& g, uint32_t w, int64_t q,
                     uint32_t flags, size_t fbudget, int32_t* d_L) {
    uint32_t ys = 0;
    while (q > 0 && (uint64_t)(q - 1) >> ys > FW<W>::kMask) ++ys;
    // q unset: buckets over a speculative range from a prefix, resolved on
    // the device into qs (the kernels read it; ys / ybase above are unused).
    const int2* qs = nullptr;
    if (SPEC) {
        const uint32_t np = (uint32_t)ctx->sm_count;
        int rc0 = chp_ensure(ctx, ctx->yrange, (size_t)(np + 1) * sizeof(int2));
        if (rc0) return rc0;
        int2* part = (int2*)ctx->yrange.p;
        k_yrange<<<np, 1024, 0, ctx->stream>>>(d_xy, std::min<uint64_t>(n, 1ull << 18), g, part);
        CHP_LAUNCHED(ctx);
        k_quant_shift<<<1, 32, 0, ctx->stream>>>(part, np, g, FW<W>::kMask, part + np);
        CHP_LAUNCHED(ctx);
        qs = part + np;
    }
    uint32_t gshift = 0;
    while ((((uint64_t)(w + (1u << gshift) - 1) >> gshift) + 1) * sizeof(W) > fbudget) ++gshift;
    const uint32_t ngroups = (w + (1u << gshift) - 1) >> gshift;
    int rc = chp_ensure(ctx, ctx->filter, (size_t)(ngroups + 1) * sizeof(W) + 16);
    if (rc) return rc;
    const Plan pl = plan_for(ctx, (size_t)(ngroups + 1) * sizeof(W), flags, false);
    // Miss handling per phase.  While the snapshots are young (phases that
    // start before n/8) misses are frequent and mostly NOT improvements, so
    // a miss reads its slot first and REDs only a real update (the REDs of
    // those phases were contended: 8 M per phase at 35-110 G/s).  Later the
    // misses are few and a read would stall the warp, so they RED one-sided
    // without reading.  C4: read-first throughout 388, RED-only 488, this
    // split 530 Gpts/s.  CHP_REDUCE_MISS_READ / _MISS_RED force one policy.
    const bool force_read = (flags & CHP_REDUCE_MISS_READ) != 0;
    const bool force_red = (flags & CHP_REDUCE_MISS_RED) != 0 && !force_read;
    const uint64_t read_until = n >> 3;
    uint64_t cur_done = 0;  // first point of the phase being launched
    auto pass = [&](const int32_t* xy, uint64_t cnt, const W* F) {
        const bool rf = force_read || (!force_red && cur_done < read_until);
        if (rf && !pl.tma) {
            auto fn = k_reduce_filter<W, true, false, SPEC>;
            CHP_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
            int per_sm = 0;
            CHP_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreadsRF, pl.smem));
            CHP_CUDA(ctx, launch_pdl(fn, dim3(std::max(1, std::min(per_sm, 2)) * ctx->sm_count), dim3(kThreadsRF),
                                     pl.smem, ctx->stream, xy, cnt, g, w, gshift, ys, F, ngroups, pl.stages, d_L,
                                     qs));
            CHP_LAUNCHED(ctx);
        } else if (rf)
            CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_filter<W, true, true, SPEC>),
                                   (k_reduce_filter<W, true, false, SPEC>), xy, cnt, g, w, gshift, ys, F, ngroups,
                                   pl.stages, d_L, qs);
        else
            CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_filter<W, false, true, SPEC>),
                                   (k_reduce_filter<W, false, false, SPEC>), xy, cnt, g, w, gshift, ys, F, ngroups,
                                   pl.stages, d_L, qs);
        return CHP_OK;
    };
    // Phases double in length: warm-up n/2^kw (default n/64) with an empty
    // table, then [d, 2d) against a snapshot of DL taken at d.  The snapshot
    // at d leaves ~1/d of the later points outside the band (SURVEY-style
    // simulation of C4: group hit rate 53% at n/64, 94% at n/7, 98% at n/2),
    // so doubling keeps the misses of every phase about equal.
    const uint32_t kfield = (flags >> 16) & 7;
    // C4 with the read-first young phases: kw 4 525, 6 537, 7 534, 9 501 Gpts/s
    const uint32_t kw = kfield ? kfield + 3 : 6;
    // (Inputs under 4 Mi points: one pass with the empty table.)
    const uint64_t warm = n < (1ull << 22) ? n : (n >> kw) & ~1ull;
    chp_trace(ctx, "filter:warm");
    if ((rc = pass(d_xy, warm, nullptr))) return rc;
    // (experiments: CHP_FILTER_YOUNG="num/den:until_shift" -- phases grow by
    // num/den until n >> until_shift, by 2 after)
    // (CHP_FILTER_SPLIT_LAST: the last phase in two halves with a rebuild
    // between, to measure what one phase boundary costs)
    struct Young {
        unsigned num = 2, den = 1, shift = 64;
        bool split_last = false;
    };
    static const Young young = [] {
        Young y;
        if (const char* e = getenv("CHP_FILTER_YOUNG")) {
            unsigned a = 2, b = 1, sh = 2;
            if (sscanf(e, "%u/%u:%u", &a, &b, &sh) == 3 && a > b && b > 0) {
                y.num = a;
                y.den = b;
                y.shift = sh;
            }
        }
        y.split_last = getenv("CHP_FILTER_SPLIT_LAST") != nullptr;
        return y;
    }();
    const uint64_t y_num = young.num, y_den = young.den, y_until = young.shift >= 64 ? 0 : n >> young.shift;
    for (uint64_t done = warm; done < n;) {
        chp_trace(ctx, "filter:build");
        CHP_CUDA(ctx, launch_pdl(k_filter_build<W>, dim3((ngroups + 1 + 255) / 256), dim3(256), 0, ctx->stream,
                                 (const int*)d_L, w, gshift, (int32_t)g.ybase, ys, (W*)ctx->filter.p, ngroups, qs));
        CHP_LAUNCHED(ctx);
        uint64_t stop = std::min<uint64_t>(n, done < y_until ? (done * y_num / y_den + 1) & ~1ull : 2 * done);
        if (young.split_last && stop == n && done >= n / 2 && n - done > (n >> 3))
            stop = (done + (n - done) / 2) & ~1ull;
        cur_done = done;
        chp_trace(ctx, "filter:phase");
        if ((rc = pass(d_xy + 2 * done, stop - done, (const W*)ctx->filter.p))) return rc;
        done = stop;
    }
    chp_trace(ctx, "filter:end");
    return CHP_OK;
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
    CHP_CUDA(ctx, launch_pdl(k_dl_init, dim3(blocks), dim3(256), 0, ctx->stream, reinterpret_cast<int4*>(d_L), n4, d_L,
                             (uint32_t)width));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

// Choice of variant: the smallest shared-memory
// footprint that holds the exact table (smem16, then smem32), else the
// column-group filter when the y range is known, else the L2 table.
// Algorithm 1 with the valid y range [ybase, ybase + ycount) (ycount < 0:
// [ybase, INT32_MAX]).  chp_reduce is ybase = 1, ycount = q; precondition
// passes the bounding box's y range, so the fast variants apply to it too.
int chp_reduce_yr(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int64_t width, int64_t ybase, int64_t ycount,
                  int64_t x_off, int32_t* d_L, uint32_t flags) {
    if (!ctx) return CHP_EINVAL;
    if (ybase < (int64_t)INT32_MIN || ybase > (int64_t)INT32_MAX) return chp_einval(ctx, "reduce: y base outside int32");
    const int64_t q = ycount;  // number of valid y values (the variants' bucket range)
    if (width < 1) return chp_einval(ctx, "reduce: width must be >= 1");
    if (width > (int64_t)INT32_MAX) return chp_einval(ctx, "reduce: width exceeds the int32 slot range");
    if ((reinterpret_cast<uintptr_t>(d_xy) & 7) || (reinterpret_cast<uintptr_t>(d_L) & 7))
        return chp_einval(ctx, "reduce: device buffers must be 8-byte aligned");
    if (x_off + 1 < (int64_t)INT32_MIN || x_off > (int64_t)INT32_MAX)
        return chp_einval(ctx, "reduce: x offset outside the int32 range");
    const bool validate = !(flags & CHP_REDUCE_NO_VALIDATE);
    const bool need_init = !(flags & CHP_REDUCE_ACCUMULATE);
    if (n == 0) return need_init ? chp_dl_init(ctx, d_L, width) : CHP_OK;

    Geo g;
    g.base = (uint32_t)(int32_t)(x_off + 1);
    const int64_t reach = (int64_t)INT32_MAX - x_off;  // x <= INT32_MAX
    g.wcheck = (uint32_t)std::min<int64_t>(width, reach);
    g.ybase = (uint32_t)(int32_t)ybase;
    g.blocked = (flags & CHP_REDUCE_BLOCKED) ? 1u : 0u;
    // number of valid y values; the host callers keep it below 2^32
    g.qmax = (uint32_t)std::min<int64_t>({q < 0 ? (int64_t)INT32_MAX - ybase + 1 : q, (int64_t)INT32_MAX - ybase + 1,
                                          (int64_t)UINT32_MAX});
    const uint32_t w = (uint32_t)width;
    const size_t budget = (size_t)std::min(ctx->smem_optin, 200 * 1024);
    const bool fits32 = (size_t)w * 8 <= budget;
    const bool y16 = validate && q >= 1 && q <= 65536;  // all valid y in [ybase, ybase + 65536)
    const bool fits16 = y16 && (size_t)w * 4 <= budget;
    const bool yknown = validate && q >= 1;  // every accepted y is in [ybase, ybase + q)
    const bool fits_f8 = yknown && ybase == 1 && (size_t)((w + 7) & ~7u) * 2 <= budget;  // quant8 assumes y >= 1

    const uint32_t wpad8 = (w + 8) & ~7u;  // >= w + 1: slot w is the invalid-x sink
    // q unset (validation y >= ybase only): the sampled filter quantises a
    // speculative range from a prefix instead (Quant, k_yrange).
    const bool yspec = validate && q < 0 && ybase >= 0;
    const bool fits_sampled = (yknown || yspec) && g.wcheck == w && (size_t)wpad8 * 2 <= budget;
    const bool fits_filter = (yknown || yspec) && g.wcheck == w;  // invalid x must clamp onto the sink

    enum { V_GLOBAL, V_SMEM32, V_SMEM16, V_FILTER8, V_FILTER, V_SAMPLED } v;
    if (flags & CHP_REDUCE_FORCE_GLOBAL) v = V_GLOBAL;
    else if ((flags & CHP_REDUCE_FORCE_SAMPLED) && fits_sampled) v = V_SAMPLED;
    else if ((flags & CHP_REDUCE_FORCE_SMEM32) && fits32) v = V_SMEM32;
    else if ((flags & CHP_REDUCE_FORCE_SMEM16) && fits16) v = V_SMEM16;
    else if ((flags & CHP_REDUCE_FORCE_FILTER8) && fits_f8) v = V_FILTER8;
    else if ((flags & CHP_REDUCE_FORCE_FILTER) && fits_filter) v = V_FILTER;
    else if (fits16) v = V_SMEM16;  // measured: 1.05-1.24x smem32 (C3, C5)
    else if (fits32) v = V_SMEM32;
    else if (fits_sampled) v = V_SAMPLED;
    else if (fits_filter) v = V_FILTER;
    else v = V_GLOBAL;

    // The sampled variant initialises DL inside its sample pass.
    if (need_init && v != V_SAMPLED) {
        int rc = chp_dl_init(ctx, d_L, width);
        if (rc) return rc;
    }

    auto launch_global = [&](const int32_t* p, uint64_t m) -> int {
        if (m == 0) return CHP_OK;
        if (flags & CHP_REDUCE_WARP_AGG) {
            auto fn = validate ? k_reduce_global_agg<true> : k_reduce_global_agg<false>;
            int blocks = 0;
            if (int rc0 = kernel_blocks(ctx, (const void*)fn, 0, 2, &blocks)) return rc0;
            fn<<<blocks, kThreads, 0, ctx->stream>>>(p, m, g, w, d_L);
            CHP_LAUNCHED(ctx);
            return CHP_OK;
        }
        const Plan pl = plan_for(ctx, 0, flags, false);
        if (validate)
            CHP_LAUNCH_PLANNED(ctx, pl, (k_reduce_global<true, true>), (k_reduce_global<true, false>), p, m, g, w,
                               pl.stages, d_L);
        else
            CHP_LAUNCH_PLANNED(ctx, pl, (k_reduce_global<false, true>), (k_reduce_global<false, false>), p, m, g, w,
                               pl.stages, d_L);
        return CHP_OK;
    };

    switch (v) {
        case V_SMEM32: {
            const Plan pl = plan_for(ctx, (size_t)w * 8, flags, true);
            if (validate)
                CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_smem32<true, true>), (k_reduce_smem32<true, false>), d_xy, n,
                                   g, w, pl.stages, d_L);
            else
                CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_smem32<false, true>), (k_reduce_smem32<false, false>), d_xy,
                                   n, g, w, pl.stages, d_L);
            ctx->variant = pl.tma ? "smem32+tma" : "smem32";
            return CHP_OK;
        }
        case V_SMEM16: {
            const Plan pl = plan_for(ctx, (size_t)w * 4, flags, false);
            // fits16 implies validation with 1 <= y <= q <= 65536 (the kernel's
            // packed window).
            CHP_LAUNCH_PLANNED_PDL(ctx, pl, k_reduce_smem16<true>, k_reduce_smem16<false>, d_xy, n, g, w, pl.stages,
                               d_L);
            ctx->variant = pl.tma ? "smem16+tma" : "smem16";
            return CHP_OK;
        }
        case V_FILTER8: {
            // Warm-up prefix through L2, per-column snapshot, learning pass.
            uint32_t ys = 0;
            while ((uint64_t)(q - 1) >> ys > 255) ++ys;
            const uint32_t wpad = (w + 7) & ~7u;
            int rc = chp_ensure(ctx, ctx->filter, (size_t)wpad * 2 + 16);
            if (rc) return rc;
            const uint64_t warm = std::min<uint64_t>(n, n / 64) & ~1ull;
            if ((rc = launch_global(d_xy, warm))) return rc;
            k_filter8_build<<<(w + 255) / 256, 256, 0, ctx->stream>>>(d_L, w, ys, (uint16_t*)ctx->filter.p);
            CHP_LAUNCHED(ctx);
            if (n > warm) {
                const Plan pl = plan_for(ctx, (size_t)wpad * 2, flags, false);
                CHP_LAUNCH_PLANNED(ctx, pl, k_reduce_filter8<true>, k_reduce_filter8<false>, d_xy + 2 * warm,
                                   n - warm, g, w, ys, (const uint16_t*)ctx->filter.p, pl.stages, d_L);
            }
            ctx->variant = "filter8";
            return CHP_OK;
        }
        case V_SAMPLED: {
            // Sample pass (n/16) -> merged strict-interior table -> one
            // pass over all n points.
            // Buckets u = umulhi(y - base, m) in [0, 254] over the q valid
            // values, monotone in y (a shift left power-of-two q at half the
            // resolution: 2^16 values -> 128 buckets of 512).  q unset: the
            // range of the valid y in the first 2^18 points, resolved on the
            // device by every consumer CTA from k_yrange's partials.
            Quant qz{(int32_t)g.ybase, yknown ? quant_mult((uint64_t)q) : quant_mult(g.qmax)};
            const int2* qpart = nullptr;
            uint32_t nqpart = 0;
            if (!yknown) {
                nqpart = (uint32_t)ctx->sm_count;
                int rc0 = chp_ensure(ctx, ctx->yrange, (size_t)nqpart * sizeof(int2));
                if (rc0) return rc0;
                qpart = (const int2*)ctx->yrange.p;
                k_yrange<<<nqpart, 1024, 0, ctx->stream>>>(d_xy, std::min<uint64_t>(n, 1ull << 18), g,
                                                            (int2*)ctx->yrange.p);
                CHP_LAUNCHED(ctx);
            }
            const size_t tbytes = (size_t)wpad8 * 2;
            const int sblocks = ctx->sm_count;
            int rc = chp_ensure(ctx, ctx->sample, (size_t)sblocks * tbytes + 16);
            if (!rc) rc = chp_ensure(ctx, ctx->filter, tbytes + 16);
            if (rc) return rc;
            // Sample = n / 2^k points, k = 4 unless CHP_REDUCE_SAMPLE_K(k): the
            // heads of the main pass's per-CTA slices, or the prefix
            // (CHP_REDUCE_SAMPLE_PREFIX).  C2, same box: n * 32/256 585-590,
            // 24/256 596, 20/256 612, 16/256 631, 14/256 638, 12/256 619,
            // 10/256 620, 8/256 600 Gpts/s (k = 3 had been best before the
            // main pass got cheaper per point).  Round 2, K1 us: 11/256 157.4,
            // 12/256 156.1, 13/256 149.5, 14/256 148.9, 15/256 148.8, 16/256
            // 149.0, 18/256 150.0 -- flat from 13/256 to 16/256.
            uint32_t f256 = 256u >> ((flags >> 16) & 7 ? (flags >> 16) & 7 : 4);
            int prefix = (flags & CHP_REDUCE_SAMPLE_PREFIX) ? 1 : 0;
            // Default: sample pass + merge as ONE cooperative kernel (a grid
            // barrier between them, the merge spread over every CTA), then the
            // main pass as a dependent launch (C2: 586 vs 573 Gpts/s for
            // separate sample / merge launches, CHP_REDUCE_SAMPLE_SPLIT).
            // CHP_REDUCE_FUSED also runs the main pass inside the same kernel
            // (slower: its main pass spills at 64 registers).
            const int merge_only = (flags & CHP_REDUCE_FUSED) ? 0 : 1;
            if (!(flags & CHP_REDUCE_SAMPLE_SPLIT) && !(flags & CHP_REDUCE_TMA) &&
                !(flags & CHP_REDUCE_SAMPLE_TMA) && ctx->coop) {
                if (!ctx->gridbar.p) {
                    if ((rc = chp_ensure(ctx, ctx->gridbar, 64))) return rc;
                    CHP_CUDA(ctx, cudaMemsetAsync(ctx->gridbar.p, 0, 64, ctx->stream));
                }
                const size_t smem = std::max(table_span(tbytes), kFusedMergeSmem);
                const void* fused = yknown ? (const void*)k_sampled_fused<false> : (const void*)k_sampled_fused<true>;
                CHP_CUDA(ctx, cudaFuncSetAttribute(fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem));
                int per_sm = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused, kThreads, smem);
                if (per_sm >= 1) {
                    const int init = need_init ? 1 : 0;
                    uint16_t* scratch = (uint16_t*)ctx->sample.p;
                    uint16_t* F = (uint16_t*)ctx->filter.p;
                    GridBar* bar = (GridBar*)ctx->gridbar.p;
                    void* args[] = {(void*)&d_xy, (void*)&n, (void*)&f256, (void*)&prefix, (void*)&g, (void*)&w, (void*)&wpad8,
                                    (void*)&qz, (void*)&qpart, (void*)&nqpart, (void*)&scratch, (void*)&F, (void*)&d_L, (void*)&init, (void*)&bar,
                                    (void*)&merge_only};
                    // (A cooperative launch can be refused when the GPU is
                    // shared and the grid cannot be co-resident: then the
                    // split form below runs instead.)
                    static const bool refuse = getenv("CHP_TEST_COOP_REFUSE") != nullptr;  // tests
                    chp_trace(ctx, "sampled:sample+merge");
                    // Cooperative AND a programmatic dependent of the
                    // previous kernel (it waits before touching DL); plain
                    // cooperative if the runtime refuses the pair.
                    cudaLaunchConfig_t lc = {};
                    lc.gridDim = dim3(sblocks * (refuse ? 64 : 1));
                    lc.blockDim = dim3(kThreads);
                    lc.dynamicSmemBytes = smem;
                    lc.stream = ctx->stream;
                    cudaLaunchAttribute la[2];
                    la[0].id = cudaLaunchAttributeCooperative;
                    la[0].val.cooperative = 1;
                    la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    la[1].val.programmaticStreamSerializationAllowed = 1;
                    lc.attrs = la;
                    lc.numAttrs = 2;
                    cudaError_t ce = cudaLaunchKernelExC(&lc, fused, args);
                    if (ce != cudaSuccess && !refuse) {
                        static bool told = false;
                        if (!told && getenv("CHP_VERBOSE")) {
                            fprintf(stderr, "chp: cooperative + programmatic launch refused (%s); cooperative only\n",
                                    cudaGetErrorString(ce));
                            told = true;
                        }
                        cudaGetLastError();
                        ce = cudaLaunchCooperativeKernel(fused, dim3(sblocks), dim3(kThreads), args, smem, ctx->stream);
                    }
                    if (ce != cudaSuccess) {
                        cudaGetLastError();
                        goto split;
                    }
                    CHP_LAUNCHED(ctx);
                    if (!merge_only) {
                        ctx->variant = yknown ? "sampled-fused" : "sampled-fused-yspec";
                        return CHP_OK;
                    }
                    const Plan pl = plan_for(ctx, tbytes, flags, false);
                    chp_trace(ctx, "sampled:main");
                    if (yknown)
                        CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_sampled<true, false>),
                                               (k_reduce_sampled<false, false>), d_xy, n, g, w, wpad8, qz, qpart,
                                               nqpart, (const uint16_t*)ctx->filter.p, pl.stages, d_L);
                    else
                        CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_sampled<true, true>), (k_reduce_sampled<false, true>),
                                               d_xy, n, g, w, wpad8, qz, qpart, nqpart,
                                               (const uint16_t*)ctx->filter.p, pl.stages, d_L);
                    ctx->variant = yknown ? "sampled" : "sampled-yspec";
                    return CHP_OK;
                }
            }
        split:
            {
                const Plan sp = plan_for(ctx, tbytes, (flags & CHP_REDUCE_SAMPLE_TMA) ? CHP_REDUCE_TMA : 0u, false);
                auto fn = sp.tma ? (yknown ? k_sample_learn<true, false> : k_sample_learn<true, true>)
                                 : (yknown ? k_sample_learn<false, false> : k_sample_learn<false, true>);
                int unused = 0;
                if ((rc = kernel_blocks(ctx, (const void*)fn, sp.smem, 1, &unused))) return rc;
                fn<<<sblocks, kThreads, sp.smem, ctx->stream>>>(d_xy, n, g, w, wpad8, qz, qpart, nqpart,
                                                                (uint16_t*)ctx->sample.p,
                                                                d_L, need_init ? 1 : 0, sp.stages, f256, prefix);
                CHP_LAUNCHED(ctx);
            }
            const uint32_t nchunks = wpad8 / 8;
            CHP_CUDA(ctx, launch_pdl(k_sample_merge, dim3((nchunks + kMergeCols - 1) / kMergeCols),
                                     dim3(kMergeCols, kMergeSlices), 0, ctx->stream,
                                     (const uint16_t*)ctx->sample.p, (uint32_t)sblocks, w, wpad8,
                                     (uint16_t*)ctx->filter.p));
            CHP_LAUNCHED(ctx);
            const Plan pl = plan_for(ctx, tbytes, flags, false);
            if (yknown)
                CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_sampled<true, false>), (k_reduce_sampled<false, false>), d_xy,
                                       n, g, w, wpad8, qz, qpart, nqpart, (const uint16_t*)ctx->filter.p, pl.stages,
                                       d_L);
            else
                CHP_LAUNCH_PLANNED_PDL(ctx, pl, (k_reduce_sampled<true, true>), (k_reduce_sampled<false, true>), d_xy,
                                       n, g, w, wpad8, qz, qpart, nqpart, (const uint16_t*)ctx->filter.p, pl.stages,
                                       d_L);
            ctx->variant = yknown ? "sampled" : "sampled-yspec";
            return CHP_OK;
        }
        case V_FILTER: {
            const size_t fbudget = (flags & CHP_REDUCE_FILTER_SMALL) ? 100 * 1024 : budget;
            int rc;
            if (flags & CHP_REDUCE_FILTER16)
                rc = yknown ? run_group_filter<uint32_t, false>(ctx, d_xy, n, g, w, q, flags, fbudget, d_L)
                            : run_group_filter<uint32_t, true>(ctx, d_xy, n, g, w, q, flags, fbudget, d_L);
            else
                rc = yknown ? run_group_filter<uint16_t, false>(ctx, d_xy, n, g, w, q, flags, fbudget, d_L)
                            : run_group_filter<uint16_t, true>(ctx, d_xy, n, g, w, q, flags, fbudget, d_L);
            if (rc) return rc;
            ctx->variant = (flags & CHP_REDUCE_FILTER16) ? (yknown ? "filter16" : "filter16-yspec")
                                                         : (yknown ? "filter" : "filter-yspec");
            return CHP_OK;
        }
        default: {
            int rc = launch_global(d_xy, n);
            if (rc) return rc;
            ctx->variant = (flags & CHP_REDUCE_WARP_AGG) ? "global-agg" : "global";
            return CHP_OK;
        }
    }
}

extern "C" int chp_reduce(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int64_t width, int64_t q,
                          int64_t x_off, int32_t* d_L, uint32_t flags) {
    return chp_reduce_yr(ctx, d_xy, n, width, 1, q, x_off, d_L, flags);
}

// Diagnostics, not part of include/chp_b200.h (tools/trace_k1.py).
extern "C" int chp_debug_trace_enable(chp_ctx* ctx, int on) {
    if (!ctx) return CHP_EINVAL;
    for (auto& t : ctx->trace) cudaEventDestroy(t.first);
    ctx->trace.clear();
    ctx->tracing = on != 0;
    return CHP_OK;
}

extern "C" int chp_debug_trace_mark(chp_ctx* ctx, const char* label) {
    if (!ctx) return CHP_EINVAL;
    chp_trace(ctx, label);
    return CHP_OK;
}

// ms[i] = time from trace point i to i + 1; labels[i] its label.  Returns the
// number of intervals written.
extern "C" int chp_debug_trace_read(chp_ctx* ctx, float* ms, const char** labels, int cap) {
    if (!ctx) return -1;
    cudaStreamSynchronize(ctx->stream);
    int k = 0;
    for (size_t i = 0; i + 1 < ctx->trace.size() && k < cap; ++i, ++k) {
        cudaEventElapsedTime(&ms[k], ctx->trace[i].first, ctx->trace[i + 1].first);
        labels[k] = ctx->trace[i].second;
    }
    return k;
}

extern "C" int chp_check(chp_ctx* ctx, const int32_t* d_L, int64_t width) {
    if (!ctx) return CHP_EINVAL;
    int32_t err = 0;
    CHP_CUDA(ctx, cudaMemcpyAsync(&err, d_L + 2 * width, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CHP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (err != 0) return chp_einval(ctx, "reduce: coordinate out of range");
    return CHP_OK;
}

#if CHP_PHASE_TIMING
extern "C" int chp_debug_phase(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_phase, sizeof(g_phase));
}
#endif
