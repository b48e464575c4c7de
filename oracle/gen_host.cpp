// gen_host.cpp -- the config 2-5 workload generators on the host, built into
// oracle/_build/libchpgen.so for the CPU legs that must not load the product
// library (bench.py --impl reference, the cpu_baseline sample).
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  It compiles the product's own
// generator header (paper_1505_00914_b200/csrc/gen.cuh: counter-based, IEEE
// basic operations only, -ffp-contract=off) for the host, so the reference
// arm consumes byte-for-byte the points the device generates
// (tests/test_oracle.py::test_host_generator_lib_matches_product).
#include <cstdint>
#include <thread>
#include <vector>

#include "gen.cuh"

extern "C" int gen_points(int config, uint64_t seed, int64_t p, uint64_t offset, uint64_t n, int32_t* xy,
                          int threads) {
    if (config < 2 || config > 5 || p < 1 || p > INT32_MAX) return 1;
    chpgen::Cluster cl[64];
    for (int c = 0; c < 64; ++c) cl[c] = chpgen::cluster_param(seed, p, c);
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n / 65536 + 1) threads = (int)(n / 65536 + 1);
    auto work = [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) chpgen::point(config, seed, p, offset + i, cl, &xy[2 * i], &xy[2 * i + 1]);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t)
        pool.emplace_back(work, n * (uint64_t)t / threads, n * (uint64_t)(t + 1) / threads);
    work(0, n / (uint64_t)threads);
    for (auto& th : pool) th.join();
    return 0;
}
