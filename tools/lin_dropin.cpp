// Replica of the reference acceptance criterion 8 timing loop (drop-in
// precondition over n = 1e5 .. 1e6 at density 0.4, min of 40 reps), with the
// per-n times printed.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "chp/reducer.hpp"

using namespace chp;

int main() {
    for (int64_t n = 100000; n <= 1000000; n += 100000) {
        const int64_t p = std::max<int64_t>(1, std::llround(std::sqrt(n / 0.4)));
        std::mt19937_64 rng(13);
        std::uniform_int_distribution<int64_t> u(1, p);
        std::vector<Point> pts(n);
        for (auto& q : pts) { q.x = u(rng); q.y = u(rng); }
        double best = 1e9, br = 1e9, be = 1e9;
        for (int r = 0; r < 40; ++r) {
            auto res = reducer::precondition(pts);
            best = std::min(best, res.total());
            br = std::min(br, res.t_reduce);
            be = std::min(be, res.t_extract);
        }
        std::printf("n=%7lld p=%5lld total=%.3f ms reduce=%.3f extract=%.3f\n", (long long)n, (long long)p, best * 1e3,
                    br * 1e3, be * 1e3);
    }
}
