// shard.cu -- Algorithm 1 over G devices in ONE process:
// the points are split into contiguous equal slices, each device folds its
// slice into a partial device-form L (DL), and the partials are combined by
// an element-wise MIN -- the DL stores (lo, ~hi) and the error word, so one
// MIN merges everything.  Exact for any partition because min and max are
// associative and commutative (the property /root/reference/proj/
// tests/test_reducer.cpp:113-127 pins; reduce itself is src/reducer.cpp:69-79).
//
// Two combines:
//   CHP_COMBINE_NCCL  ncclAllReduce(ncclInt32, ncclMin) over the group's
//                     communicator (ncclCommInitAll over the G devices);
//                     NVLink/NVSwitch on an 8 x B200 box.  libnccl.so.2 is
//                     loaded on first use, so the library itself does not
//                     depend on NCCL.
//   CHP_COMBINE_PEER  device 0 waits for every partial (stream events) and
//                     ONE kernel reads the G partial DLs over peer memory
//                     (P2P loads through NVLink) into DL 0.  Devices may
//                     repeat: G contexts on one device run the same code path
//                     (how the 1-GPU test box exercises G > 1).
//   CHP_COMBINE_FUSED no partial DLs and no combine step: device 0
//                     initialises DL 0 and every shard's K1 folds straight
//                     into it over peer memory (its flush and miss-path REDs
//                     are NVLink atomics on device 0's L2), so the exchange
//                     happens inside K1, overlapped with the other shards'
//                     streams.  Best where K1 touches L little (shared-memory
//                     tables flushed once per CTA: C5's 256 columns); every
//                     L2 access of a filter variant becomes remote.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "chp_internal.cuh"

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        a.commInitAll = (decltype(a.commInitAll))dlsym(h, "ncclCommInitAll");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
        a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
        a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
        a.errStr = (decltype(a.errStr))dlsym(h, "ncclGetErrorString");
        a.ok = a.commInitAll && a.commDestroy && a.allReduce && a.groupStart && a.groupEnd && a.errStr;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

constexpr int kMaxShards = 16;

struct PeerDL {
    const int2* p[kMaxShards];
};

// out[i] = min over g of in[g][i], per 32-bit word (pairs (lo, ~hi), error
// word, pad).  in[0] may alias out.
__global__ void k_dl_min_peers(PeerDL in, int G, uint64_t n2, int2* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
        int2 m = in.p[0][i];
        for (int g = 1; g < G; ++g) {
            const int2 v = in.p[g][i];
            m.x = min(m.x, v.x);
            m.y = min(m.y, v.y);
        }
        out[i] = m;
    }
}

}  // namespace

struct chp_group {
    int G = 0;
    int combine = CHP_COMBINE_NCCL;
    std::vector<int> dev;
    std::vector<chp_ctx*> ctx;
    std::vector<ncclComm_t> comm;
    std::vector<cudaEvent_t> folded;  // per shard: its partial DL is complete
    cudaEvent_t combined = nullptr;   // (peer) the combine kernel has read every partial;
                                      // (fused) DL 0 is initialised
    std::string err;
    uint64_t h2d_bytes = 0;
};

namespace {

int gfail(chp_group* g, int rc, const std::string& msg) {
    g->err = msg;
    return rc;
}

int gctx_fail(chp_group* g, int k, int rc) {
    return gfail(g, rc, "shard " + std::to_string(k) + ": " + chp_last_error(g->ctx[k]));
}

// Contiguous equal slices: shard k owns [k n / G, (k + 1) n / G).
void slice(uint64_t n, int G, int k, uint64_t* lo, uint64_t* cnt) {
    const unsigned __int128 a = (unsigned __int128)n * (unsigned)k / (unsigned)G;
    const unsigned __int128 b = (unsigned __int128)n * (unsigned)(k + 1) / (unsigned)G;
    *lo = (uint64_t)a;
    *cnt = (uint64_t)(b - a);
}

// Merge the partial DLs d_L[0..G) so that d_L[0] (NCCL: every d_L[k]) holds
// the element-wise MIN.  Stream-ordered after each shard's K1.
int combine(chp_group* g, int32_t* const* d_L, int64_t width) {
    const uint64_t words = chp_dl_len(width);
    if (g->G == 1 && g->combine != CHP_COMBINE_NCCL) return CHP_OK;
    if (g->combine == CHP_COMBINE_FUSED) {  // DL 0 already holds everything: device 0 waits for the shards
        for (int k = 1; k < g->G; ++k) {
            cudaSetDevice(g->dev[k]);
            if (cudaEventRecord(g->folded[k], g->ctx[k]->stream) != cudaSuccess)
                return gfail(g, CHP_EDEVICE, "cudaEventRecord");
        }
        cudaSetDevice(g->dev[0]);
        for (int k = 1; k < g->G; ++k)
            if (cudaStreamWaitEvent(g->ctx[0]->stream, g->folded[k], 0) != cudaSuccess)
                return gfail(g, CHP_EDEVICE, "cudaStreamWaitEvent");
        return CHP_OK;
    }
    if (g->combine == CHP_COMBINE_NCCL) {
        const NcclApi& api = nccl();
        ncclResult_t r = api.groupStart();
        for (int k = 0; k < g->G && r == ncclSuccess; ++k) {
            cudaSetDevice(g->dev[k]);
            r = api.allReduce(d_L[k], d_L[k], words, ncclInt32, ncclMin, g->comm[k], g->ctx[k]->stream);
        }
        const ncclResult_t r2 = api.groupEnd();
        if (r == ncclSuccess) r = r2;
        if (r != ncclSuccess) return gfail(g, CHP_EDEVICE, std::string("ncclAllReduce: ") + api.errStr(r));
        return CHP_OK;
    }
    chp_ctx* c0 = g->ctx[0];
    for (int k = 1; k < g->G; ++k) {
        cudaSetDevice(g->dev[k]);
        if (cudaEventRecord(g->folded[k], g->ctx[k]->stream) != cudaSuccess)
            return gfail(g, CHP_EDEVICE, "cudaEventRecord");
    }
    cudaSetDevice(g->dev[0]);
    for (int k = 1; k < g->G; ++k)
        if (cudaStreamWaitEvent(c0->stream, g->folded[k], 0) != cudaSuccess)
            return gfail(g, CHP_EDEVICE, "cudaStreamWaitEvent");
    PeerDL in;
    for (int k = 0; k < g->G; ++k) in.p[k] = reinterpret_cast<const int2*>(d_L[k]);
    const uint64_t n2 = words / 2;
    const int blocks = (int)std::min<uint64_t>((n2 + 255) / 256, (uint64_t)c0->sm_count * 4);
    k_dl_min_peers<<<std::max(blocks, 1), 256, 0, c0->stream>>>(in, g->G, n2, reinterpret_cast<int2*>(d_L[0]));
    c0->launches++;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gfail(g, CHP_EDEVICE, std::string("k_dl_min_peers: ") + cudaGetErrorString(e));
    // Later work on a shard's stream (the next call's DL init) must not
    // overwrite its partial while the combine still reads it.
    if (cudaEventRecord(g->combined, c0->stream) != cudaSuccess) return gfail(g, CHP_EDEVICE, "cudaEventRecord");
    for (int k = 1; k < g->G; ++k) {
        cudaSetDevice(g->dev[k]);
        if (cudaStreamWaitEvent(g->ctx[k]->stream, g->combined, 0) != cudaSuccess)
            return gfail(g, CHP_EDEVICE, "cudaStreamWaitEvent");
    }
    return CHP_OK;
}

// The caller's current device, restored on exit (the group calls switch
// between the shards' devices).
struct DeviceGuard {
    int dev = 0;
    DeviceGuard() { cudaGetDevice(&dev); }
    ~DeviceGuard() { cudaSetDevice(dev); }
};

// CHP_COMBINE_FUSED: DL 0 initialised on device 0, every shard stream
// ordered after it.
int fused_init(chp_group* g, int32_t* dl0, int64_t width) {
    cudaSetDevice(g->dev[0]);
    int rc = chp_dl_init(g->ctx[0], dl0, width);
    if (rc) return gctx_fail(g, 0, rc);
    if (cudaEventRecord(g->combined, g->ctx[0]->stream) != cudaSuccess) return gfail(g, CHP_EDEVICE, "cudaEventRecord");
    for (int k = 1; k < g->G; ++k) {
        cudaSetDevice(g->dev[k]);
        if (cudaStreamWaitEvent(g->ctx[k]->stream, g->combined, 0) != cudaSuccess)
            return gfail(g, CHP_EDEVICE, "cudaStreamWaitEvent");
    }
    return CHP_OK;
}

template <typename T>
int pipeline_sharded(chp_group* g, const T* h_xy, uint64_t n, int64_t width, int64_t q, int32_t* h_Lpairs,
                     uint64_t* h_occ, int32_t* h_chain, int64_t* h_s, int32_t* h_hull, int64_t* h_h) {
    if (!g) return CHP_EINVAL;
    DeviceGuard keep;
    g->h2d_bytes = 0;
    if (width < 1) return gfail(g, CHP_EINVAL, "reduce: width must be >= 1");
    if (width > (1ll << 29)) return gfail(g, CHP_EINVAL, "reduce: width exceeds the device limit 2^29");
    std::vector<int32_t*> dl(g->G);
    const bool fused = g->combine == CHP_COMBINE_FUSED;
    for (int k = 0; k < g->G; ++k) {
        chp_ctx* c = g->ctx[k];
        cudaSetDevice(c->device);
        if (fused && k > 0) {  // every shard folds into shard 0's DL
            dl[k] = dl[0];
            continue;
        }
        const int rc = chp_ensure(c, c->dl, chp_dl_len(width) * 4);
        if (rc) return gctx_fail(g, k, rc);
        dl[k] = (int32_t*)c->dl.p;
    }
    if (fused) {
        const int rc = fused_init(g, dl[0], width);
        if (rc) return rc;
    }
    // One host thread per shard: each streams its slice (chunked H2D, packed
    // where the range allows) into its device's partial DL.
    std::vector<int> rcs(g->G, CHP_OK);
    auto work = [&](int k) {
        uint64_t lo, cnt;
        slice(n, g->G, k, &lo, &cnt);
        if constexpr (sizeof(T) == 4)
            rcs[k] = fused ? chp_reduce_host_into(g->ctx[k], h_xy + 2 * lo, cnt, width, q, dl[k])
                           : chp_reduce_host(g->ctx[k], h_xy + 2 * lo, cnt, width, q, dl[k]);
        else
            rcs[k] = fused ? chp_reduce_host64_into(g->ctx[k], h_xy + 2 * lo, cnt, width, q, dl[k])
                           : chp_reduce_host64(g->ctx[k], h_xy + 2 * lo, cnt, width, q, dl[k]);
    };
    std::vector<std::thread> th;
    for (int k = 1; k < g->G; ++k) th.emplace_back(work, k);
    work(0);
    for (auto& t : th) t.join();
    for (int k = 0; k < g->G; ++k) {
        if (rcs[k]) return gctx_fail(g, k, rcs[k]);
        g->h2d_bytes += chp_last_h2d_bytes(g->ctx[k]);
    }
    int rc = combine(g, dl.data(), width);
    if (rc) return rc;
    rc = chp_finish_host(g->ctx[0], dl[0], width, h_Lpairs, h_occ, h_chain, h_s, h_hull, h_h);
    if (rc) return gctx_fail(g, 0, rc);
    return CHP_OK;
}

}  // namespace

extern "C" {

int chp_group_create(const int* devices, int G, int combine_mode, chp_group** out) {
    if (!out) return CHP_EINVAL;
    DeviceGuard keep;
    *out = nullptr;
    if (!devices || G < 1 || G > kMaxShards) return CHP_EINVAL;
    if (combine_mode != CHP_COMBINE_NCCL && combine_mode != CHP_COMBINE_PEER && combine_mode != CHP_COMBINE_FUSED)
        return CHP_EINVAL;
    chp_group* g = new chp_group();
    g->G = G;
    g->combine = combine_mode;
    g->dev.assign(devices, devices + G);
    auto bail = [&](int rc) {
        chp_group_destroy(g);
        return rc;
    };
    if (combine_mode == CHP_COMBINE_NCCL) {
        for (int a = 0; a < G; ++a)
            for (int b = a + 1; b < G; ++b)
                if (devices[a] == devices[b]) return bail(CHP_EINVAL);  // NCCL: one rank per device
    }
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    for (int k = 0; k < G; ++k) {
        chp_ctx* c = nullptr;
        if (chp_ctx_create(devices[k], &c) != CHP_OK) return bail(CHP_EDEVICE);
        // the shards' host packing pools share the host cores
        c->pool_parts = (int)std::max(2u, std::min(hw, 32u) / (unsigned)G);
        g->ctx.push_back(c);
    }
    if (combine_mode != CHP_COMBINE_NCCL) {  // peer or fused: events and peer access to device 0
        g->folded.resize(G, nullptr);
        for (int k = 0; k < G; ++k) {
            cudaSetDevice(devices[k]);
            if (cudaEventCreateWithFlags(&g->folded[k], cudaEventDisableTiming) != cudaSuccess)
                return bail(CHP_EDEVICE);
        }
        // peer: device 0 reads every partial DL; fused: every device
        // reads and REDs device 0's DL
        cudaSetDevice(devices[0]);
        if (cudaEventCreateWithFlags(&g->combined, cudaEventDisableTiming) != cudaSuccess) return bail(CHP_EDEVICE);
        for (int k = 1; k < G; ++k) {
            if (devices[k] == devices[0]) continue;
            const int from = combine_mode == CHP_COMBINE_PEER ? devices[0] : devices[k];
            const int to = combine_mode == CHP_COMBINE_PEER ? devices[k] : devices[0];
            int can = 0;
            cudaDeviceCanAccessPeer(&can, from, to);
            if (!can) return bail(CHP_EDEVICE);
            cudaSetDevice(from);
            const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return bail(CHP_EDEVICE);
            cudaGetLastError();
        }
    } else {
        const NcclApi& api = nccl();
        if (!api.ok) return bail(CHP_EDEVICE);
        g->comm.resize(G, nullptr);
        if (api.commInitAll(g->comm.data(), G, devices) != ncclSuccess) {
            g->comm.clear();
            return bail(CHP_EDEVICE);
        }
    }
    *out = g;
    return CHP_OK;
}

void chp_group_destroy(chp_group* g) {
    if (!g) return;
    DeviceGuard keep;
    for (int k = 0; k < (int)g->ctx.size(); ++k) chp_ctx_sync(g->ctx[k]);
    if (!g->comm.empty()) {
        const NcclApi& api = nccl();
        for (ncclComm_t c : g->comm)
            if (c) api.commDestroy(c);
    }
    for (size_t k = 0; k < g->folded.size(); ++k)
        if (g->folded[k]) {
            cudaSetDevice(g->dev[k]);
            cudaEventDestroy(g->folded[k]);
        }
    if (g->combined) {
        cudaSetDevice(g->dev[0]);
        cudaEventDestroy(g->combined);
    }
    for (chp_ctx* c : g->ctx) chp_ctx_destroy(c);
    delete g;
}

chp_ctx* chp_group_ctx(chp_group* g, int k) { return (g && k >= 0 && k < g->G) ? g->ctx[k] : nullptr; }

int chp_group_size(const chp_group* g) { return g ? g->G : 0; }

const char* chp_group_last_error(const chp_group* g) { return g ? g->err.c_str() : "null group"; }

uint64_t chp_group_last_h2d_bytes(const chp_group* g) { return g ? g->h2d_bytes : 0; }

int chp_reduce_sharded(chp_group* g, const int32_t* const* d_xy, const uint64_t* n, int64_t width, int64_t q,
                       int32_t* const* d_L) {
    if (!g || !d_xy || !n || !d_L) return CHP_EINVAL;
    DeviceGuard keep;
    const bool fused = g->combine == CHP_COMBINE_FUSED;
    if (fused) {
        if (width < 1 || width > (int64_t)INT32_MAX) return gfail(g, CHP_EINVAL, "reduce: width out of range");
        int rc = fused_init(g, d_L[0], width);
        if (rc) return rc;
    }
    for (int k = 0; k < g->G; ++k) {
        cudaSetDevice(g->dev[k]);
        const int rc = fused ? chp_reduce(g->ctx[k], d_xy[k], n[k], width, q, 0, d_L[0], CHP_REDUCE_ACCUMULATE)
                             : chp_reduce(g->ctx[k], d_xy[k], n[k], width, q, 0, d_L[k], 0);
        if (rc) return gctx_fail(g, k, rc);
    }
    return combine(g, d_L, width);
}

int chp_pipeline_host_sharded(chp_group* g, const int32_t* h_xy, uint64_t n, int64_t width, int64_t q,
                              int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s, int32_t* h_hull,
                              int64_t* h_h) {
    return pipeline_sharded(g, h_xy, n, width, q, h_Lpairs, h_occ, h_chain, h_s, h_hull, h_h);
}

int chp_pipeline_host64_sharded(chp_group* g, const int64_t* h_xy, uint64_t n, int64_t width, int64_t q,
                                int32_t* h_Lpairs, uint64_t* h_occ, int32_t* h_chain, int64_t* h_s,
                                int32_t* h_hull, int64_t* h_h) {
    return pipeline_sharded(g, h_xy, n, width, q, h_Lpairs, h_occ, h_chain, h_s, h_hull, h_h);
}

}  // extern "C"
