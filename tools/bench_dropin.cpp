// End-to-end time of the C++ drop-in as a reference user calls it: int64
// Points in a std::vector, reducer::reduce + build_polyline (width known),
// and reducer::precondition (width unknown), on C2-shaped data (argv[2] = 5:
// C5-shaped, 90% of x in 4 columns of 256, y uniform in [1, 256]).
// g++ -std=c++20 -O2 -Iinclude tools/bench_dropin.cpp -Lpaper_1505_00914_b200/lib -lchp_b200 \
//     -Wl,-rpath,'$ORIGIN/../paper_1505_00914_b200/lib' -o tools/bench_dropin
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <random>
#include <vector>

#include "chp/reducer.hpp"

using namespace chp;

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::stoull(argv[1]) : 100000000ull;
    const int cfg = argc > 2 ? std::atoi(argv[2]) : 2;
    const int64_t P = cfg == 5 ? 256 : 65536;
    std::vector<Point> pts(n);
    std::mt19937_64 rng(2);
    std::normal_distribution<double> nd(32768.0, 8192.0);
    std::uniform_int_distribution<int64_t> u(1, P), hot(127, 130), coin(0, 9);
    for (auto& p : pts) {
        if (cfg == 5) {
            p.x = coin(rng) ? hot(rng) : u(rng);
            p.y = u(rng);
        } else {
            p.x = std::min<int64_t>(65536, std::max<int64_t>(1, std::llround(nd(rng))));
            p.y = std::min<int64_t>(65536, std::max<int64_t>(1, std::llround(nd(rng))));
        }
    }
    auto time = [&](const char* what, auto&& f) {
        f();  // warm-up
        double best = 1e9;
        for (int r = 0; r < 3; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            f();
            best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        std::printf("%-40s %8.1f ms  %6.2f Gpts/s\n", what, best * 1e3, n / best / 1e9);
    };
    size_t s = 0;
    time("reduce(q=p) + build_polyline", [&] {
        auto arr = reducer::reduce(pts, P, P);
        s = reducer::build_polyline(arr).vertices.size();
    });
    time("reduce(q unset) + build_polyline", [&] {
        auto arr = reducer::reduce(pts, P);
        s = reducer::build_polyline(arr).vertices.size();
    });
    time("precondition", [&] { s = reducer::precondition(pts).chain.vertices.size(); });
    std::printf("chain length %zu\n", s);
    return 0;
}
