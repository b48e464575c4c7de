// gen.cuh -- deterministic synthetic workloads for BASELINE.json configs 2-5.
//
// Point i of a stream is a pure function of (config, seed, p, i): a
// counter-based splitmix64 draw per (i, k) and only IEEE-754 basic
// operations (+ - * / sqrt, floor), which are correctly rounded on both the
// host (x86-64 SSE2, -ffp-contract=off) and the device (explicit __d*_rn
// intrinsics, so nvcc cannot contract to FMA).  The host and device
// therefore emit identical bytes, so the CPU oracle and the GPU consume the
// same input without copying 8-32 GB across PCIe.  The natural logarithm the
// Gaussian needs is computed with a fixed atanh series (det_log) for the
// same reason: libm and CUDA's log() are not guaranteed to agree.
#pragma once
#include <cstdint>
#include <cstring>
#include <cmath>

#ifdef __CUDACC__
#define CHP_HD __host__ __device__ __forceinline__
#else
#define CHP_HD inline
#endif

namespace chpgen {

CHP_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
CHP_HD double dsub(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
CHP_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
CHP_HD double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
CHP_HD double dsqrt(double a) {
#ifdef __CUDA_ARCH__
    return __dsqrt_rn(a);
#else
    return std::sqrt(a);
#endif
}
CHP_HD double dfloor(double a) {
#ifdef __CUDA_ARCH__
    return ::floor(a);
#else
    return std::floor(a);
#endif
}
CHP_HD uint64_t mulhi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}
CHP_HD uint64_t dbits(double d) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
#endif
}
CHP_HD double bitsd(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double d;
    std::memcpy(&d, &u, 8);
    return d;
#endif
}

// splitmix64 finaliser.
CHP_HD uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Draw k of point i on the stream keyed by `key`.
CHP_HD uint64_t draw(uint64_t key, uint64_t i, uint64_t k) {
    return mix64(mix64(key + i * 0x9E3779B97F4A7C15ull) ^ (k * 0xD1B54A32D192ED03ull + 0x8CB92BA72F3D8DD7ull));
}

CHP_HD uint64_t stream_key(uint64_t seed, uint64_t config) {
    return mix64(seed * 0xA0761D6478BD642Full + config * 0xE7037ED1A0B428DBull + 0x1234567ull);
}

// Uniform double in [0,1) with 53 random bits.
CHP_HD double unit(uint64_t r) { return dmul((double)(r >> 11), 1.1102230246251565e-16); /* 2^-53 */ }

// Uniform integer in [1,p].
CHP_HD int64_t uniform1(uint64_t r, int64_t p) { return 1 + (int64_t)mulhi(r, (uint64_t)p); }

// Round half away from zero (std::llround semantics) and clamp to [1,p].
CHP_HD int32_t round_clamp(double v, int64_t p) {
    double r = v >= 0.0 ? dfloor(dadd(v, 0.5)) : -dfloor(dadd(-v, 0.5));
    if (r < 1.0) return 1;
    if (r > (double)p) return (int32_t)p;
    return (int32_t)(int64_t)r;
}

// ln(s) for s in (0, 1]: s = m 2^e, m in [sqrt(1/2), sqrt(2)), then
// ln m = 2 atanh t, t = (m-1)/(m+1), |t| <= 0.1716, series to t^23.
CHP_HD double det_log(double s) {
    uint64_t b = dbits(s);
    int e = (int)((b >> 52) & 0x7FF) - 1023;
    double m = bitsd((b & 0x000FFFFFFFFFFFFFull) | (1023ull << 52));
    if (m > 1.4142135623730951) {
        m = dmul(m, 0.5);
        e += 1;
    }
    const double t = ddiv(dsub(m, 1.0), dadd(m, 1.0));
    const double t2 = dmul(t, t);
    double sum = ddiv(1.0, 23.0);
    for (int k = 21; k >= 1; k -= 2) sum = dadd(dmul(sum, t2), ddiv(1.0, (double)k));
    return dadd(dmul(dmul(2.0, t), sum), dmul((double)e, 0.6931471805599453));
}

// Marsaglia polar method: two independent N(0,1) from draws k0, k0+1, ...
// Returns the next unused draw index.
CHP_HD uint64_t polar(uint64_t key, uint64_t i, uint64_t k, double* z1, double* z2) {
    for (;;) {
        const double u = dsub(dmul(2.0, unit(draw(key, i, k))), 1.0);
        const double v = dsub(dmul(2.0, unit(draw(key, i, k + 1))), 1.0);
        k += 2;
        const double s = dadd(dmul(u, u), dmul(v, v));
        if (s > 0.0 && s < 1.0) {
            const double f = dsqrt(ddiv(dmul(-2.0, det_log(s)), s));
            *z1 = dmul(u, f);
            *z2 = dmul(v, f);
            return k;
        }
    }
}

// Config-4 cluster parameters (64 clusters): centre uniform in [1,p]^2,
// sd uniform in [p/512, p/32].
struct Cluster {
    double cx, cy, sd;
};
CHP_HD Cluster cluster_param(uint64_t seed, int64_t p, int c) {
    const uint64_t key = stream_key(seed, 104);
    const double pd = (double)p;
    Cluster cl;
    cl.cx = dadd(1.0, dmul(dsub(pd, 1.0), unit(draw(key, (uint64_t)c, 0))));
    cl.cy = dadd(1.0, dmul(dsub(pd, 1.0), unit(draw(key, (uint64_t)c, 1))));
    const double lo = ddiv(pd, 512.0), hi = ddiv(pd, 32.0);
    cl.sd = dadd(lo, dmul(dsub(hi, lo), unit(draw(key, (uint64_t)c, 2))));
    return cl;
}

// Point i of config `cfg`.  Returns false for an unknown config.
CHP_HD bool point(int cfg, uint64_t seed, int64_t p, uint64_t i, const Cluster* clusters,
                  int32_t* x, int32_t* y) {
    const uint64_t key = stream_key(seed, (uint64_t)cfg);
    const double pd = (double)p;
    switch (cfg) {
        case 2: {  // x,y iid N(p/2, (p/8)^2), rounded, clamped to [1,p]
            double z1, z2;
            polar(key, i, 0, &z1, &z2);
            const double mu = dmul(pd, 0.5), sd = dmul(pd, 0.125);
            *x = round_clamp(dadd(mu, dmul(sd, z1)), p);
            *y = round_clamp(dadd(mu, dmul(sd, z2)), p);
            return true;
        }
        case 3: {  // area-uniform in the inscribed disk, by rejection
            const double r = dmul(pd, 0.5);
            for (uint64_t k = 0;; k += 2) {
                const double u = dsub(dmul(2.0, unit(draw(key, i, k))), 1.0);
                const double v = dsub(dmul(2.0, unit(draw(key, i, k + 1))), 1.0);
                if (dadd(dmul(u, u), dmul(v, v)) < 1.0) {
                    *x = round_clamp(dadd(r, dmul(r, u)), p);
                    *y = round_clamp(dadd(r, dmul(r, v)), p);
                    return true;
                }
            }
        }
        case 4: {  // 99%: 64 equal-weight isotropic Gaussians; 1%: uniform
            const uint64_t r0 = draw(key, i, 0);
            if (r0 < 184467440737095516ull) {  // floor(0.01 * 2^64)
                *x = (int32_t)uniform1(draw(key, i, 1), p);
                *y = (int32_t)uniform1(draw(key, i, 2), p);
                return true;
            }
            const int c = (int)mulhi(draw(key, i, 1), 64);
            double z1, z2;
            polar(key, i, 2, &z1, &z2);
            const Cluster cl = clusters[c];
            *x = round_clamp(dadd(cl.cx, dmul(cl.sd, z1)), p);
            *y = round_clamp(dadd(cl.cy, dmul(cl.sd, z2)), p);
            return true;
        }
        case 5: {  // 90%: x in the 4 adjacent columns p/2-1 .. p/2+2; 10%: uniform
            const uint64_t r0 = draw(key, i, 0);
            if (r0 < 16602069666338596454ull) {  // floor(0.9 * 2^64)
                const int64_t base = p / 2 - 1 < 1 ? 1 : p / 2 - 1;
                int64_t xx = base + (int64_t)mulhi(draw(key, i, 1), 4);
                *x = (int32_t)(xx > p ? p : xx);
            } else {
                *x = (int32_t)uniform1(draw(key, i, 1), p);
            }
            *y = (int32_t)uniform1(draw(key, i, 2), p);
            return true;
        }
        default:
            return false;
    }
}

}  // namespace chpgen
