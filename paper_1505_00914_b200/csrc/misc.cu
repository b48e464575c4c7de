// misc.cu -- K0 bounds, translation and the synthetic workload generators.
//
// chp_bounds replaces kernels::min_max / min_max_avx2
// (/root/reference/proj/src/kernels.cpp:55-58, src/kernels_avx2.cpp:25-53):
// one streaming pass, warp shuffles, one atomic per warp.  chp_translate
// replaces kernels::translate (src/kernels.cpp:60-65); on the hot path the
// translation is fused into K1's slot computation instead (x_off).
#include <algorithm>
#include <thread>
#include <vector>

#include "chp_internal.cuh"
#include "gen.cuh"

namespace {

__global__ void k_bounds_init(int* out4) {
    out4[0] = INT_MAX;
    out4[1] = INT_MIN;
    out4[2] = INT_MAX;
    out4[3] = INT_MIN;
}

__global__ void __launch_bounds__(512) k_bounds(const int32_t* __restrict__ xy, uint64_t n, int* __restrict__ out4) {
    int xmin = INT_MAX, xmax = INT_MIN, ymin = INT_MAX, ymax = INT_MIN;
    const bool head = (reinterpret_cast<uintptr_t>(xy) & 15) != 0;
    const uint64_t h = head ? 1 : 0;
    const uint64_t nvec = (n - h) / 2;
    const int4* v = reinterpret_cast<const int4*>(xy + 2 * h);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    auto f = [&](int x, int y) {
        xmin = min(xmin, x);
        xmax = max(xmax, x);
        ymin = min(ymin, y);
        ymax = max(ymax, y);
    };
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nvec; i += 4 * stride) {
        const int4 a = ld_stream(v + i), b = ld_stream(v + i + stride);
        const int4 c = ld_stream(v + i + 2 * stride), d = ld_stream(v + i + 3 * stride);
        f(a.x, a.y); f(a.z, a.w); f(b.x, b.y); f(b.z, b.w);
        f(c.x, c.y); f(c.z, c.w); f(d.x, d.y); f(d.z, d.w);
    }
    for (; i < nvec; i += stride) {
        const int4 a = ld_stream(v + i);
        f(a.x, a.y);
        f(a.z, a.w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (head) f(xy[0], xy[1]);
        if ((n - h) & 1) f(xy[2 * (n - 1)], xy[2 * (n - 1) + 1]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        xmin = min(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
        xmax = max(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
        ymin = min(ymin, __shfl_xor_sync(0xffffffffu, ymin, o));
        ymax = max(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
    }
    // Block reduction, then one atomic per word per block (per-warp atomics
    // on four addresses serialised at L2: 28 us for 1 M points).
    __shared__ int red[4][16];
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][warp] = xmin;
        red[1][warp] = xmax;
        red[2][warp] = ymin;
        red[3][warp] = ymax;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        int a = l < nw ? red[0][l] : INT_MAX, b = l < nw ? red[1][l] : INT_MIN;
        int c = l < nw ? red[2][l] : INT_MAX, d = l < nw ? red[3][l] : INT_MIN;
        for (int o = 8; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
            c = min(c, __shfl_xor_sync(0xffffffffu, c, o));
            d = max(d, __shfl_xor_sync(0xffffffffu, d, o));
        }
        if (l == 0) {
            atomicMin(out4 + 0, a);
            atomicMax(out4 + 1, b);
            atomicMin(out4 + 2, c);
            atomicMax(out4 + 3, d);
        }
    }
}

__global__ void k_translate(const int2* __restrict__ in, uint64_t n, int dx, int dy, int2* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int2 p = in[i];
        out[i] = make_int2((int)((unsigned)p.x + (unsigned)dx), (int)((unsigned)p.y + (unsigned)dy));
    }
}

__global__ void k_dl_from_pairs(const int2* __restrict__ pairs, uint64_t width, int2* __restrict__ DL) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < width; i += stride) {
        const int2 e = pairs[i];
        DL[i] = e.x <= e.y ? make_int2(e.x, ~e.y) : make_int2(CHP_EMPTY, CHP_EMPTY);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) DL[width] = make_int2(0, 0);
}

struct Clusters {
    chpgen::Cluster c[64];
};

__global__ void k_generate(int cfg, uint64_t seed, int64_t p, uint64_t offset, uint64_t n, Clusters cl,
                           int2* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int32_t x, y;
        chpgen::point(cfg, seed, p, offset + i, cl.c, &x, &y);
        out[i] = make_int2(x, y);
    }
}

Clusters make_clusters(uint64_t seed, int64_t p) {
    Clusters cl;
    for (int c = 0; c < 64; ++c) cl.c[c] = chpgen::cluster_param(seed, p, c);
    return cl;
}

}  // namespace

namespace {
// Four packed points (one 16-byte load) -> two 16-byte stores.
__global__ void k_unpack16(const uint4* __restrict__ in4, uint64_t n4, const uint32_t* __restrict__ in, uint64_t n,
                           int32_t base, int32_t ybase, int4* __restrict__ out4, int2* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 q = __ldcs(in4 + i);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        int v[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = (int)(w[k] & 0xFFFFu) + base;
            v[2 * k + 1] = (int)(w[k] >> 16) + ybase;
        }
        out4[2 * i] = make_int4(v[0], v[1], v[2], v[3]);
        out4[2 * i + 1] = make_int4(v[4], v[5], v[6], v[7]);
    }
    if (blockIdx.x == 0)
        for (uint64_t i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x)
            out[i] = make_int2((int)(in[i] & 0xFFFFu) + base, (int)(in[i] >> 16) + ybase);
}
// 42-bit form for ranges up to 2^21 x 2^21: point v = slot | (y - ybase) << 21,
// three per 16-byte word: lo64 = v0 | v1 << 42, hi64 = v1 >> 22 | v2 << 20.
__global__ void k_unpack42(const uint4* __restrict__ in, uint64_t n, int32_t base, int32_t ybase,
                           int2* __restrict__ out) {
    const uint64_t nw = (n + 2) / 3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr uint64_t M21 = (1ull << 21) - 1, M42 = (1ull << 42) - 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += stride) {
        const uint4 q = __ldcs(in + i);
        const uint64_t lo = (uint64_t)q.x | ((uint64_t)q.y << 32), hi = (uint64_t)q.z | ((uint64_t)q.w << 32);
        const uint64_t v[3] = {lo & M42, (lo >> 42) | ((hi << 22) & M42), hi >> 20};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint64_t j = 3 * i + k;
            if (j < n) out[j] = make_int2((int)(uint32_t)(v[k] & M21) + base, (int)(uint32_t)(v[k] >> 21) + ybase);
        }
    }
}
// 16-bit form for ranges up to 2^8 x 2^8: point v = slot | (y - ybase) << 8,
// eight per 16-byte word -> four 16-byte stores.
__global__ void k_unpack8(const uint4* __restrict__ in8, uint64_t n, int32_t base, int32_t ybase,
                          int4* __restrict__ out4, int2* __restrict__ out, int vec) {
    const uint64_t nw = n / 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += stride) {
        const uint4 q = __ldcs(in8 + i);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        int v[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[4 * k] = (int)(w[k] & 0xFFu) + base;
            v[4 * k + 1] = (int)((w[k] >> 8) & 0xFFu) + ybase;
            v[4 * k + 2] = (int)((w[k] >> 16) & 0xFFu) + base;
            v[4 * k + 3] = (int)(w[k] >> 24) + ybase;
        }
        if (vec) {
#pragma unroll
            for (int k = 0; k < 4; ++k) out4[4 * i + k] = make_int4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) out[8 * i + k] = make_int2(v[2 * k], v[2 * k + 1]);
        }
    }
    if (blockIdx.x == 0) {
        const uint16_t* in16 = reinterpret_cast<const uint16_t*>(in8);
        for (uint64_t j = 8 * nw + threadIdx.x; j < n; j += blockDim.x) {
            CHP_CHECK(j < n && j / 8 == nw);
            out[j] = make_int2((int)(in16[j] & 0xFFu) + base, (int)(in16[j] >> 8) + ybase);
        }
    }
}
}  // namespace

int chp_unpack8(chp_ctx* ctx, const void* d_in, uint64_t n, int32_t base, int32_t ybase, int32_t* d_out) {
    if (n == 0) return CHP_OK;
    const uint64_t nw = n / 8;
    const int vec = (reinterpret_cast<uintptr_t>(d_out) & 15) == 0;
    const int blocks = (int)std::min<uint64_t>((nw + 255) / 256 + 1, (uint64_t)ctx->sm_count * 8);
    k_unpack8<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const uint4*>(d_in), n, base, ybase,
                                               reinterpret_cast<int4*>(d_out), reinterpret_cast<int2*>(d_out), vec);
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

int chp_unpack42(chp_ctx* ctx, const void* d_in, uint64_t n, int32_t base, int32_t ybase, int32_t* d_out) {
    if (n == 0) return CHP_OK;
    const uint64_t nw = (n + 2) / 3;
    const int blocks = (int)std::min<uint64_t>((nw + 255) / 256, (uint64_t)ctx->sm_count * 8);
    k_unpack42<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const uint4*>(d_in), n, base, ybase,
                                                reinterpret_cast<int2*>(d_out));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

int chp_unpack16(chp_ctx* ctx, const uint32_t* d_in, uint64_t n, int32_t base, int32_t ybase, int32_t* d_out) {
    if (n == 0) return CHP_OK;
    const bool vec = !(reinterpret_cast<uintptr_t>(d_in) & 15) && !(reinterpret_cast<uintptr_t>(d_out) & 15);
    const uint64_t n4 = vec ? n / 4 : 0;
    const int blocks = (int)std::min<uint64_t>((n4 + 255) / 256 + 1, (uint64_t)ctx->sm_count * 8);
    k_unpack16<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const uint4*>(d_in), n4, d_in, n, base, ybase,
                                                reinterpret_cast<int4*>(d_out), reinterpret_cast<int2*>(d_out));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

int chp_bounds_init(chp_ctx* ctx, int32_t* d_out4) {
    k_bounds_init<<<1, 1, 0, ctx->stream>>>(d_out4);
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

int chp_bounds_accumulate(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int32_t* d_out4) {
    if (n == 0) return CHP_OK;
    const int blocks = (int)std::min<uint64_t>((n / 2 + 511) / 512 + 1, (uint64_t)ctx->sm_count * 4);
    k_bounds<<<blocks, 512, 0, ctx->stream>>>(d_xy, n, d_out4);
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

extern "C" int chp_bounds(chp_ctx* ctx, const int32_t* d_xy, uint64_t n, int32_t* d_out4) {
    if (!ctx) return CHP_EINVAL;
    if (n == 0) return chp_einval(ctx, "min_max: empty input");
    int rc = chp_bounds_init(ctx, d_out4);
    if (rc) return rc;
    return chp_bounds_accumulate(ctx, d_xy, n, d_out4);
}

extern "C" int chp_translate(chp_ctx* ctx, const int32_t* d_in, uint64_t n, int32_t dx, int32_t dy,
                             int32_t* d_out) {
    if (!ctx) return CHP_EINVAL;
    if (n == 0) return CHP_OK;
    const int blocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sm_count * 16);
    k_translate<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const int2*>(d_in), n, dx, dy,
                                                 reinterpret_cast<int2*>(d_out));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

extern "C" int chp_dl_from_pairs(chp_ctx* ctx, const int32_t* d_Lpairs, int64_t width, int32_t* d_L) {
    if (!ctx) return CHP_EINVAL;
    if (width < 1) return chp_einval(ctx, "dl_from_pairs: width must be >= 1");
    const int blocks = (int)std::min<uint64_t>(((uint64_t)width + 255) / 256, (uint64_t)ctx->sm_count * 16);
    k_dl_from_pairs<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const int2*>(d_Lpairs), (uint64_t)width,
                                                     reinterpret_cast<int2*>(d_L));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

extern "C" int chp_generate(chp_ctx* ctx, int config, uint64_t seed, int64_t p, uint64_t offset, uint64_t n,
                            int32_t* d_xy) {
    if (!ctx) return CHP_EINVAL;
    if (config < 2 || config > 5) return chp_einval(ctx, "generate: device configs are 2..5");
    if (p < 1 || p > INT32_MAX) return chp_einval(ctx, "generate: p out of range");
    if (n == 0) return CHP_OK;
    const Clusters cl = make_clusters(seed, p);
    const int blocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sm_count * 32);
    k_generate<<<blocks, 256, 0, ctx->stream>>>(config, seed, p, offset, n, cl, reinterpret_cast<int2*>(d_xy));
    CHP_LAUNCHED(ctx);
    return CHP_OK;
}

extern "C" int chp_generate_host(int config, uint64_t seed, int64_t p, uint64_t offset, uint64_t n,
                                 int32_t* h_xy, int threads) {
    if (config < 2 || config > 5 || p < 1 || p > INT32_MAX) return CHP_EINVAL;
    const Clusters cl = make_clusters(seed, p);
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n / 65536 + 1) threads = (int)(n / 65536 + 1);
    auto work = [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i)
            chpgen::point(config, seed, p, offset + i, cl.c, &h_xy[2 * i], &h_xy[2 * i + 1]);
    };
    if (threads == 1) {
        work(0, n);
        return CHP_OK;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back(work, n * (uint64_t)t / threads, n * (uint64_t)(t + 1) / threads);
    for (auto& th : pool) th.join();
    return CHP_OK;
}
