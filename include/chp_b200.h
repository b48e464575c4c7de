/*
 * chp_b200.h -- C ABI of the B200 (sm_100a) hot path of the convex-hull
 * preconditioner (arXiv 1505.00914, Algorithm 1 + Lemma-1 compaction + hull).
 *
 * Plain C: POD arguments, device pointers are plain `int32_t*` etc., no torch
 * or CUDA types in any signature (streams travel as `void*`).  Every call is
 * stream-ordered on the context's stream; functions that return results to
 * the host say so.  One context per device per host thread; contexts are not
 * thread-safe, different contexts are independent.
 *
 * Status codes: CHP_OK; CHP_EINVAL where the reference throws
 * std::invalid_argument; CHP_EDEVICE for CUDA failures (the C++ drop-in maps
 * it to std::runtime_error).  chp_last_error() describes the last failure.
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/proj):
 *   chp_reduce            chp::reducer::reduce          include/chp/reducer.hpp:65-67,
 *                                                       src/reducer.cpp:69-79 (+ bucket :19-32)
 *   chp_compact           chp::reducer::build_polyline  include/chp/reducer.hpp:76, src/reducer.cpp:108-119;
 *                         ExtremalArray::valid_count    src/reducer.cpp:42-49;
 *                         occupancy::BlockedBitset words include/chp/occupancy.hpp:58-109;
 *                         serialize's (width+1,-1) form  src/reducer.cpp:121-130
 *   chp_ns_chain          the north_star chain order (no reference function)
 *   chp_hull              chp::hulls::melkman           include/chp/hulls.hpp:24, src/hulls.cpp:137-181
 *                         + canonicalize_hull           src/geometry.cpp:42-80
 *   chp_bounds            chp::kernels::min_max         include/chp/kernels.hpp:33, src/kernels.cpp:55-58
 *   chp_translate         chp::kernels::translate       include/chp/kernels.hpp:34-35, src/kernels.cpp:60-65
 *   chp_pipeline_host     reduce + build_polyline (+ melkman) from HOST buffers, the drop-in's
 *                         workhorse (src/reducer.cpp:69-79, :108-119; src/hulls.cpp:137-181)
 *   chp_reduce_host /     the two halves of chp_pipeline_host (reduce into a device L;
 *   chp_finish_host       build_polyline + melkman of it), for cross-device combines
 *   chp_reduce_sharded,   chp::reducer::reduce over G devices: no reference
 *   chp_pipeline_host_sharded  counterpart (the reference is single-threaded); same L as
 *                         src/reducer.cpp:69-79, merge law tests/test_reducer.cpp:113-127
 *   chp_precondition_host chp::reducer::precondition    include/chp/reducer.hpp:100-101,
 *   chp_precondition_run  (one-pass form of the above, outputs via chp_last_outputs)
 *                                                       src/reducer.cpp:132-178
 */
#ifndef CHP_B200_H
#define CHP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHP_OK 0
#define CHP_EINVAL 1
#define CHP_EDEVICE 2

typedef struct chp_ctx chp_ctx;

/* ---------------------------------------------------------------- context */
int chp_ctx_create(int device, chp_ctx** out);
void chp_ctx_destroy(chp_ctx* ctx);
const char* chp_last_error(const chp_ctx* ctx);
/* Run on a caller-owned cudaStream_t (e.g. torch's current stream); NULL is
 * the legacy default stream.  chp_ctx_use_own_stream() switches back to the
 * context's own non-blocking stream (the initial state).  A switch orders
 * the new stream after all work the context issued on the old one (the
 * context's scratch is shared by its calls), so one context's calls never
 * overlap, whatever streams they are issued on. */
int chp_ctx_set_stream(chp_ctx* ctx, void* cuda_stream);
int chp_ctx_use_own_stream(chp_ctx* ctx);
void* chp_ctx_stream(const chp_ctx* ctx);
int chp_ctx_sync(chp_ctx* ctx);
/* Number of kernels this context has launched (evidence for the bench). */
uint64_t chp_launch_count(const chp_ctx* ctx);
/* Kernel-variant name chosen by the last chp_reduce ("smem32", "smem16",
 * "global", "filter"). */
const char* chp_last_variant(const chp_ctx* ctx);
/* Host->device bytes the last host pipeline call (chp_*_host) copied: 8 per
 * point as int32 pairs, 4 per point when the input was packed to 16 bits. */
uint64_t chp_last_h2d_bytes(const chp_ctx* ctx);

/* ------------------------------------------------- device-form L ("DL")
 * int32[chp_dl_len(width)] = width pairs (lo, ~hi), empty = (INT32_MAX,
 * INT32_MAX), then the error word (0 ok, -1 = an out-of-range coordinate
 * was seen), then one pad word.  Every word is min-combined, so partial DLs
 * from several devices merge with one element-wise MIN all-reduce. */
uint64_t chp_dl_len(int64_t width);

/* ------------------------------------------------------- K1: reduction */
#define CHP_REDUCE_ACCUMULATE 1u   /* do not initialise d_L first            */
#define CHP_REDUCE_NO_VALIDATE 2u  /* precondition path: y is not checked    */
#define CHP_REDUCE_FORCE_GLOBAL 4u /* testing: force the global-L variant    */
#define CHP_REDUCE_FORCE_SMEM32 8u /* testing: force 8-byte smem slots       */
#define CHP_REDUCE_FORCE_FILTER 16u /* testing: force the column-group filter  */
#define CHP_REDUCE_FORCE_FILTER8 32u /* testing: force the per-column filter   */
#define CHP_REDUCE_FORCE_SMEM16 64u /* testing: force 4-byte packed smem slots */
#define CHP_REDUCE_MISS_RED 128u    /* tuning: filter misses always RED without reading */
#define CHP_REDUCE_MISS_READ 256u   /* tuning: filter misses always read the slot first */
#define CHP_REDUCE_FILTER16 512u    /* tuning: 16-bit filter halves (default 8) */
#define CHP_REDUCE_FILTER_SMALL 1024u /* tuning: filter table <= 100 KB (default 200 KB) */
#define CHP_REDUCE_NO_TMA 2048u     /* tuning: stream via registers, not the TMA ring */
#define CHP_REDUCE_TMA 4096u        /* tuning: stream via the TMA bulk-copy ring */
#define CHP_REDUCE_FORCE_SAMPLED 8192u /* testing: force the sampled per-column filter */
#define CHP_REDUCE_FUSED 16384u     /* tuning: sampled filter as 1 cooperative kernel (grid barriers) */
#define CHP_REDUCE_SAMPLE_K(k) ((uint32_t)(k) << 16) /* tuning (k in 1..7): the sampled filter samples n/2^k
                                                         (default 4); the group filter warms up on n/2^(k+3)
                                                         (default 6) */
#define CHP_REDUCE_SAMPLE_TMA (1u << 22) /* tuning: sample pass streams through the TMA ring */
#define CHP_PIPELINE_NO_PACK (1u << 23) /* host pipelines: always send int32 pairs (no 16/42-bit packing) */
#define CHP_REDUCE_SAMPLE_SPLIT (1u << 25) /* tuning: sampled filter's sample pass and merge as separate launches */
#define CHP_REDUCE_BLOCKED (1u << 26) /* tuning: smem/filter streams in per-CTA contiguous slices (the sampled main pass always is) */
#define CHP_REDUCE_SAMPLE_PREFIX (1u << 27) /* tuning: sampled filter samples the first n/2^k points (default: the head of each CTA slice) */
#define CHP_REDUCE_WARP_AGG (1u << 28) /* global variant: warp-aggregated updates (__match_any_sync + __reduce_min_sync,
                                          one read-compare-RED per distinct slot per warp) */

/* Algorithm 1 over n int32 (x,y) pairs at d_xy (8-byte aligned).  Slot of a
 * point is x - x_off - 1; a point is valid when that slot is in [0,width)
 * and (unless NO_VALIDATE) 1 <= y <= q (q < 0: no upper bound; the filter
 * variants then bucket a y range taken from a prefix, exact for any y).
 * Invalid points are skipped and flagged in d_L's error word; chp_check()
 * turns the flag into CHP_EINVAL.  Asynchronous (no host synchronisation). */
int chp_reduce(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int64_t width,
               int64_t q, int64_t x_off, int32_t* d_L, uint32_t flags);

/* Initialise d_L to all-empty / no-error.  Asynchronous. */
int chp_dl_init(chp_ctx* ctx, int32_t* d_L, int64_t width);

/* Rebuild a DL from (lo,hi) pairs in serialize form (empty = any lo > hi,
 * e.g. the (width+1,-1) sentinel).  Used when a caller hands back a host
 * ExtremalArray (build_polyline on an array it built or edited).  Async. */
int chp_dl_from_pairs(chp_ctx* ctx, const int32_t* d_Lpairs, int64_t width,
                      int32_t* d_L);

/* Synchronise and read d_L's error word: CHP_EINVAL if an invalid
 * coordinate was seen (reference: std::invalid_argument,
 * src/reducer.cpp:72-75). */
int chp_check(chp_ctx* ctx, const int32_t* d_L, int64_t width);

/* ------------------------------------------------------ K3: compaction
 * Single-pass decoupled-look-back scan over the slots of d_L.  All output
 * pointers are optional (NULL = not produced):
 *   d_chain  : int32 (x,y)[<= 2*width]  Lemma-1 order: per valid slot
 *              ascending, to_original(i,lo) then to_original(i,hi) if hi!=lo
 *   d_occ    : uint64[ceil(width/64)]   BlockedBitset<uint64_t> words
 *   d_Lpairs : int32 (lo,hi)[width]     empty slots as (width+1,-1)
 *   d_lower  : int32 (major,lo+minor_off)[v]  valid slots ascending
 *   d_upper  : int32 (major,hi+minor_off)[v]  valid slots ascending
 *   d_upperd : int32 (major,hi+minor_off)[s-v] slots with hi!=lo ascending
 * d_counts (required, int64[4]) receives {s, v, err, s-v}: chain length
 * (= valid_count), valid slots, the error word, two-point slots.  The
 * mapping is ExtremalArray::to_original (include/chp/reducer.hpp:46-50):
 * original = (slot + major_off, value + minor_off), axes swapped back when
 * `swapped`.  width <= 2^29.  Asynchronous. */
int chp_compact(chp_ctx* ctx, const int32_t* d_L, int64_t width,
                int64_t major_off, int64_t minor_off, int swapped,
                int32_t* d_chain, uint64_t* d_occ, int32_t* d_Lpairs,
                int32_t* d_lower, int32_t* d_upper, int32_t* d_upperd,
                int64_t* d_counts);

/* The north_star order from chp_compact's d_lower/d_upperd/d_counts: minima
 * by increasing x, then maxima (hi != lo only) by decreasing x.  d_ns has
 * room for 2*width points.  Asynchronous. */
int chp_ns_chain(chp_ctx* ctx, const int32_t* d_lower, const int32_t* d_upperd,
                 const int64_t* d_counts, int64_t width, int32_t* d_ns);

/* ------------------------------------------------------------- K4: hull
 * Exact strict convex hull of the reduced set from chp_compact's
 * d_lower / d_upper / d_counts, canonical like canonicalize_hull: CCW,
 * starting at the lexicographically smallest vertex, 1 or 2 vertices when
 * degenerate.  d_hull has room for 2*width+2 points; *d_h receives h
 * (device int64).  `swapped` as in chp_compact.  Asynchronous. */
int chp_hull(chp_ctx* ctx, const int32_t* d_lower, const int32_t* d_upper,
             const int64_t* d_counts, int64_t width, int swapped,
             int32_t* d_hull, int64_t* d_h);

/* --------------------------------------------------- K0: bounds/translate */
/* out4 (device int32[4]) = {x_min, x_max, y_min, y_max}; n >= 1. */
int chp_bounds(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int32_t* d_out4);
/* out[i] = in[i] + (dx, dy); in and out may alias. */
int chp_translate(chp_ctx* ctx, const int32_t* d_in, uint64_t n, int32_t dx,
                  int32_t dy, int32_t* d_out);

/* translate on HOST buffers (kernels::translate): H2D, kernel, D2H. */
int chp_translate_host(chp_ctx* ctx, const int32_t* h_in, uint64_t n, int32_t dx,
                       int32_t dy, int32_t* h_out);

/* ------------------------------------------------ host-buffer pipelines
 * Inputs and outputs in HOST memory; pinned inputs are copied directly,
 * pageable ones through the context's pinned staging.  The copy of chunk
 * k+1 overlaps the reduction of chunk k.  All outputs optional; synchronous;
 * CHP_EINVAL on an out-of-range coordinate (reduce) or an empty chain when a
 * chain / hull was requested (build_polyline, melkman). */
int chp_pipeline_host(chp_ctx* ctx, const int32_t* h_xy, uint64_t n,
                      int64_t width, int64_t q, int32_t* h_Lpairs,
                      uint64_t* h_occ, int32_t* h_chain, int64_t* h_s,
                      int32_t* h_hull, int64_t* h_h);

/* build_polyline / valid_count of a HOST L in serialize form (h_Lpairs,
 * empty slots any lo > hi) with ExtremalArray's offsets: uploads L, K3 on
 * device, chain back.  h_chain holds 2*width points.  CHP_EINVAL when no
 * slot is valid and h_chain is requested (src/reducer.cpp:116-117). */
int chp_polyline_host(chp_ctx* ctx, const int32_t* h_Lpairs, int64_t width,
                      int64_t major_off, int64_t minor_off, int swapped,
                      int32_t* h_chain, int64_t* h_s);

/* The two halves of chp_pipeline_host, for callers that combine partial Ls
 * across devices between them (bench.py's N > 1 e2e leg, shard groups):
 * chp_reduce_host initialises the caller's device DL d_L and streams the
 * HOST points into it (chunked H2D overlapped with K1, packed where the
 * range allows); it returns once the host buffer is no longer read and d_L
 * is complete, WITHOUT failing on an invalid coordinate (the error word
 * travels in d_L, so it survives a MIN combine).  chp_finish_host compacts
 * a device DL (K3, + K4 when a hull is requested) and copies the requested
 * outputs to the host, CHP_EINVAL when the error word is set (as
 * chp_pipeline_host).  Both synchronous. */
int chp_reduce_host(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int64_t width, int64_t q, int32_t* d_L);
int chp_reduce_host64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q, int32_t* d_L);
int chp_finish_host(chp_ctx* ctx, const int32_t* d_L, int64_t width, int32_t* h_Lpairs, uint64_t* h_occ,
                    int32_t* h_chain, int64_t* h_s, int32_t* h_hull, int64_t* h_h);

/* precondition (x-only mode, src/reducer.cpp:132-178): bounds, width =
 * x_max-x_min+1, fold with x_off = x_min-1 and y untranslated, Lemma-1
 * chain.  h_bbox4 = {x_min,x_max,y_min,y_max}.  The chain buffer must hold
 * 2*width points: call with h_chain == NULL first to learn width via
 * h_bbox4.  n >= 1 (else CHP_EINVAL). */
int chp_precondition_host(chp_ctx* ctx, const int32_t* h_xy, uint64_t n,
                          int64_t* h_bbox4, int32_t* h_Lpairs, int32_t* h_chain,
                          int64_t* h_s, int32_t* h_hull, int64_t* h_h);

/* The same in ONE pass over the input when the width is not known up
 * front: bounds, K1, K3 (and K4 when want_hull) run and the results stay
 * on the device; *h_width, *h_s (chain length) and *h_h (hull size) tell
 * the caller how much to allocate, then chp_last_outputs copies them out
 * (h_Lpairs: width pairs, h_chain: s points, h_hull: h points; any may be
 * NULL).  The results stay valid until the next host call on the context. */
int chp_precondition_run(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int want_hull,
                         int64_t* h_bbox4, int64_t* h_width, int64_t* h_s, int64_t* h_h);
int chp_last_outputs(chp_ctx* ctx, int32_t* h_Lpairs, int32_t* h_chain, int32_t* h_hull);

/* int64 forms for callers holding the reference's Point {int64 x, y}
 * (the C++ drop-in): the host pool narrows or packs straight from the int64
 * pairs (a coordinate outside int32 is CHP_EINVAL), no int32 copy first.
 * chp_precondition_run64 with swap_axes reads (y, x).  chp_bounds_host64 is
 * kernels::min_max: K0 on the device over the narrowed points. */
int chp_pipeline_host64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q,
                        int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s,
                        int32_t* h_hull, int64_t* h_h);
int chp_precondition_run64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int swap_axes, int want_hull,
                           int64_t* h_bbox4, int64_t* h_width, int64_t* h_s, int64_t* h_h);
int chp_bounds_host64(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t* h_bbox4);

/* ------------------------------------------- multi-GPU shard groups
 * reduce over G devices of one box in ONE process: the
 * points are split into contiguous equal slices (shard k owns
 * [k n/G, (k+1) n/G)), each device folds its slice into a partial DL, and
 * the partials meet in ONE element-wise MIN (storing ~hi makes every DL
 * word a min; the error word merges too).  Exact for any partition: the
 * same L as src/reducer.cpp:69-79 over all n points (min/max are
 * associative and commutative, tests/test_reducer.cpp:113-127).
 *   CHP_COMBINE_NCCL  ncclAllReduce(ncclInt32, ncclMin) over a communicator
 *                     from ncclCommInitAll (distinct devices; libnccl.so.2
 *                     is loaded on first use)
 *   CHP_COMBINE_PEER  device 0 waits on every shard's K1 and one kernel
 *                     reads the partial DLs over peer memory (NVLink P2P);
 *                     devices may repeat (G contexts on one device).
 *   CHP_COMBINE_FUSED every shard's K1 folds straight into device 0's DL
 *                     over peer memory (NVLink atomics), no combine step;
 *                     only d_L[0] is used; devices may repeat. */
#define CHP_COMBINE_NCCL 0
#define CHP_COMBINE_PEER 1
#define CHP_COMBINE_FUSED 2
typedef struct chp_group chp_group;
int chp_group_create(const int* devices, int G, int combine, chp_group** out);
void chp_group_destroy(chp_group* g);
/* The context of shard k (owned by the group; usable for single-device calls). */
chp_ctx* chp_group_ctx(chp_group* g, int k);
int chp_group_size(const chp_group* g);
const char* chp_group_last_error(const chp_group* g);
/* Host->device bytes of the last chp_pipeline_host*_sharded call, all shards. */
uint64_t chp_group_last_h2d_bytes(const chp_group* g);
/* Device-resident shards: d_xy[k] (n[k] points) on shard k's device.  On
 * return (asynchronous, on the shards' context streams) d_L[0] holds the
 * merged DL -- with CHP_COMBINE_NCCL every d_L[k] does.  Compact it with
 * chp_compact on chp_group_ctx(g, 0).  Later work on any shard's stream is
 * ordered after the combine (CHP_COMBINE_PEER: each shard stream waits for
 * the combine kernel's reads of its partial).  The group calls leave the
 * caller's current device unchanged. */
int chp_reduce_sharded(chp_group* g, const int32_t* const* d_xy, const uint64_t* n, int64_t width, int64_t q,
                       int32_t* const* d_L);
/* chp_pipeline_host over the group: one host thread per shard streams its
 * slice of the HOST input to its device, the partial DLs are combined, and
 * K3 (+K4) run on shard 0; outputs and errors exactly as chp_pipeline_host
 * (the int64 form as chp_pipeline_host64).  Synchronous. */
int chp_pipeline_host_sharded(chp_group* g, const int32_t* h_xy, uint64_t n, int64_t width, int64_t q,
                              int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s,
                              int32_t* h_hull, int64_t* h_h);
int chp_pipeline_host64_sharded(chp_group* g, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q,
                                int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s,
                                int32_t* h_hull, int64_t* h_h);

/* ------------------------------------------------- synthetic workloads
 * Deterministic, counter-based generators of the BASELINE.json configs
 * (DESIGN.md "Workloads"); identical bytes on host and device.  config:
 * 2 Gaussian, 3 disk, 4 clusters, 5 hot columns (point i of the stream is
 * a pure function of (config, seed, p, offset+i)).  Config 1 is the
 * reference's own sequential uniform-box generator (std::mt19937_64,
 * src/dataset.cpp:35-59) and exists on the host only. */
int chp_generate(chp_ctx* ctx, int config, uint64_t seed, int64_t p,
                 uint64_t offset, uint64_t n, int32_t* d_xy);
int chp_generate_host(int config, uint64_t seed, int64_t p, uint64_t offset,
                      uint64_t n, int32_t* h_xy, int threads);

#ifdef __cplusplus
}
#endif
#endif /* CHP_B200_H */
