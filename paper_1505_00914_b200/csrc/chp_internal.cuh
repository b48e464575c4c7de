// chp_internal.cuh -- context, launch bookkeeping and device helpers shared
// by the sm_100a kernels behind include/chp_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstdint>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "chp_b200.h"

#define CHP_EMPTY INT_MAX  // lo and ~hi of an empty slot

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct chp_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host pipeline: H2D overlapped with K1
    int sm_count = 148;
    int smem_optin = 227 * 1024;
    int l2_bytes = 0;
    uint64_t launches = 0;
    std::string err;
    const char* variant = "none";
    // scratch owned by the context
    DevBuf tile_status;  // K3 look-back status words: two arrays, used alternately
    uint32_t status_cap = 0, status_clean[2] = {0, 0}, compact_resident = 0;
    int compact_form = 0;  // K3 tile shape the resident count was taken for
    int status_parity = 0;
    DevBuf hull_a, hull_b, hull_cnt_a, hull_cnt_b;
    DevBuf filter;       // K1 filter snapshot
    DevBuf sample;       // K1 sampled filter: per-CTA learned tables
    DevBuf gridbar;      // grid barrier of the cooperative sampled kernel
    DevBuf yrange;       // K1 sampled filter, q unset: per-CTA y range of a prefix
    int coop = 0;        // cudaDevAttrCooperativeLaunch
    int hull_coop_checked = 0, hull_coop_ok = 0, hull_leaf_attr = 0, hull_small_attr = 0;  // K4 launch shape (hull.cu)
    DevBuf dl;           // host pipeline: device-form L
    DevBuf counts;       // host pipeline: int64[8]
    DevBuf chain, lower, upper, hull, occ, lpairs;
    DevBuf stage_dev[2]; // host pipeline: device input chunks
    void* stage_host[2] = {nullptr, nullptr};  // pinned staging for pageable inputs
    size_t stage_bytes = 0;
    cudaEvent_t ev_switch = nullptr;  // chp_ctx_set_stream: the old stream's work before the new one's
    cudaEvent_t ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_consumed[2] = {nullptr, nullptr};
    // Packed host pipeline: pinned 4-byte/point staging, unpacked device
    // chunks, and a persistent host thread pool (abi.cu HostPool).
    void* pack_host[2] = {nullptr, nullptr};
    size_t pack_bytes = 0;
    DevBuf unpack_dev[2];
    void* pool = nullptr;
    int pool_parts = 0;      // host threads of the pool (0: all cores, <= 32); shard groups split the cores
    uint64_t h2d_bytes = 0;  // of the current / last host pipeline call
    // Hybrid packed pipeline: int32 chunks DMA'd straight from a pinned input
    // while the host packs (abi.cu), and the measured host pack rate.
    DevBuf raw_dev[2];
    DevBuf points;  // precondition: the resident input (bounds, then K1)
    // chp_precondition_run's results, held on device until chp_last_outputs
    bool last_valid = false;
    int64_t last_width = 0, last_s = 0, last_h = -1;
    cudaEvent_t ev_rcopied[2] = {nullptr, nullptr};
    cudaEvent_t ev_rconsumed[2] = {nullptr, nullptr};
    double pack_rate = 8e9;    // points / s, 16-bit packing
    double pack_rate42 = 6e9;  // points / s, 42-bit packing
    double pack_rate8 = 8e9;   // points / s, 8-bit packing
    // Launch-setup cache (reduce.cu kernel_blocks): kernel -> (dynamic smem
    // it was configured for, resident blocks per SM at that size).
    std::unordered_map<const void*, std::pair<size_t, int>> kcache;
    // Diagnostics (chp_debug_trace_*; not in the header): an event recorded
    // on the stream at each traced point of K1's launch sequence.
    bool tracing = false;
    std::vector<std::pair<cudaEvent_t, const char*>> trace;
};

static inline void chp_trace(chp_ctx* ctx, const char* what) {
    if (!ctx->tracing) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, ctx->stream);
    ctx->trace.emplace_back(e, what);
}

// Record the first CUDA error of a launch sequence in ctx->err.
static inline int chp_cuda_fail(chp_ctx* ctx, cudaError_t e, const char* what) {
    ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
    return CHP_EDEVICE;
}
#define CHP_CUDA(ctx, call)                                                 \
    do {                                                                    \
        cudaError_t e_ = (call);                                            \
        if (e_ != cudaSuccess) return chp_cuda_fail((ctx), e_, #call);      \
    } while (0)
#define CHP_LAUNCHED(ctx)                                                   \
    do {                                                                    \
        (ctx)->launches++;                                                  \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) return chp_cuda_fail((ctx), e_, "kernel launch"); \
    } while (0)

static inline int chp_einval(chp_ctx* ctx, const char* msg) {
    ctx->err = msg;
    return CHP_EINVAL;
}

// Grow-only device scratch.
static inline int chp_ensure(chp_ctx* ctx, DevBuf& b, size_t bytes) {
    if (b.bytes >= bytes) return CHP_OK;
    if (b.p) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
    }
    size_t want = bytes < 256 ? 256 : bytes;
    CHP_CUDA(ctx, cudaMalloc(&b.p, want));
    b.bytes = want;
    return CHP_OK;
}

// Host points folded into an initialised DL (abi.cu; shard groups'
// CHP_COMBINE_FUSED, where the DL is shard 0's, read and REDed over peer
// memory by the other devices).  extern "C" linkage, not in the header.
extern "C" int chp_reduce_host_into(chp_ctx* ctx, const int32_t* h_xy, uint64_t n, int64_t width, int64_t q,
                                    int32_t* d_L);
extern "C" int chp_reduce_host64_into(chp_ctx* ctx, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q,
                                      int32_t* d_L);

// K0 pieces used by the host pipelines (misc.cu).
int chp_bounds_init(chp_ctx* ctx, int32_t* d_out4);
int chp_bounds_accumulate(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int32_t* d_out4);
// Packed host pipeline (abi.cu): 32-bit words (slot | (y - 1) << 16) back to
// int32 (x, y) pairs with x = slot + base.
int chp_unpack16(chp_ctx* ctx, const uint32_t* d_in, uint64_t n, int32_t base, int32_t ybase, int32_t* d_out);
// The same for 16-bit points (slot | (y - ybase) << 8), eight per 16-byte word.
int chp_unpack8(chp_ctx* ctx, const void* d_in, uint64_t n, int32_t base, int32_t ybase, int32_t* d_out);
// The same for 42-bit points (slot | (y - ybase) << 21), three per 16-byte word.
int chp_unpack42(chp_ctx* ctx, const void* d_in, uint64_t n, int32_t base, int32_t ybase, int32_t* d_out);
// K1 with a general valid y range [ybase, ybase + ycount) (reduce.cu).
int chp_reduce_yr(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int64_t width, int64_t ybase, int64_t ycount,
                  int64_t x_off, int32_t* d_L, uint32_t flags);

// ----------------------------------------------------------- device side

// Diagnostics build (CHP_NVCC_EXTRA=-DCHP_BOUNDS=1, CHP_LIB_VARIANT=bounds):
// index checks on the output writes of the kernels that trap on failure --
// compute-sanitizer is not available on the test pool.
#ifndef CHP_BOUNDS
#define CHP_BOUNDS 0
#endif
#define CHP_CHECK(cond)                                                              \
    do {                                                                             \
        if (CHP_BOUNDS && !(cond)) {                                                 \
            printf("chp bounds check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
            __trap();                                                                \
        }                                                                            \
    } while (0)

// 128-bit streaming load: read-only path, no L1 allocation, 256-byte L2
// sector prefetch (the point stream is touched exactly once, sequentially).
__device__ __forceinline__ int4 ld_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
// Grid-wide barrier of a cooperative launch (every CTA co-resident).  Each
// launch starts with count == 0 and leaves it 0: after its LAST barrier
// every CTA calls grid_barrier_done(), and the final one to do so resets
// the words (no CTA polls the counter any more by then).  A launch that is
// refused never touches the words; two cooperative kernels of one context
// never overlap (chp_ctx_set_stream orders the context's streams).  So no
// launch depends on another's grid size or barrier count.
struct GridBar {
    unsigned long long count;  // arrivals in the current launch
    unsigned long long exits;  // CTAs past their last barrier
};

__device__ __forceinline__ void grid_barrier(GridBar* b) {
    // One atomic per CTA: arrival k of barrier round r sees old = r * G + k,
    // and the round is complete once the counter reaches (r + 1) * G.  The
    // last arrival's add releases everyone directly (the reset-and-flip form
    // needed two more serialised L2 round trips, ~2 us at 148 CTAs).
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long G = gridDim.x;
        const unsigned long long old = atomicAdd(&b->count, 1ull);
        const unsigned long long target = old - old % G + G;
        unsigned long long cur;
        // Relaxed polls (an acquire load invalidates L1 on every poll:
        // CCTL.IVALL), then one fence that orders the reads after the
        // barrier behind the observed arrivals.
        do {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(&b->count) : "memory");
        } while (cur < target);
        __threadfence();
    }
    __syncthreads();
}

// After a CTA's last grid_barrier of the launch (thread 0 has observed the
// release, so it no longer reads the counter).
__device__ __forceinline__ void grid_barrier_done(GridBar* b) {
    if (threadIdx.x == 0) {
        const unsigned long long old = atomicAdd(&b->exits, 1ull);
        if (old == gridDim.x - 1ull) {
            atomicExch(&b->count, 0ull);
            atomicExch(&b->exits, 0ull);
        }
    }
}

// L2-coherent load of a slot pair that other CTAs update atomically.
__device__ __forceinline__ int2 ld_cg2(const int2* p) {
    int2 r;
    asm volatile("ld.global.cg.v2.s32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
// Fire-and-forget global min (SASS RED.MIN).
// Programmatic dependent launch.  A kernel launched with launch_pdl may be
// scheduled while its predecessor on the stream is still running; it must
// call pdl_wait() before touching anything the predecessor writes (the wait
// returns once that grid has completed and its writes are visible; it is a
// no-op without the launch attribute).  pdl_trigger() lets the dependent be
// scheduled before this grid ends.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ void red_min(int* p, int v) {
    asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Slot of x for offset x_off, as an unsigned value that is < width exactly
// when x - x_off - 1 is in [0, width).  Computed mod 2^32 (x_off + 1 fits
// int32 whenever a valid point exists).
__device__ __forceinline__ uint32_t slot_of(int32_t x, uint32_t base) {
    return (uint32_t)x - base;
}
