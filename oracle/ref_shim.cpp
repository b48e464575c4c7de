// ref_shim.cpp -- extern "C" entry points over the REFERENCE library itself.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources, where they lie under
// /root/reference/proj/src, into oracle/_ref/libchpref.so.  Nothing here
// re-implements the algorithm: every call goes to chp::reducer / chp::hulls /
// chp::dataset.  Used (a) by tests/test_oracle.py to pin the C restatement
// in chp_oracle.c against the real reference, and (b) by bench.py's
// cpu_baseline and --impl reference legs to time the reference on the host.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <optional>
#include <thread>
#include <vector>

#include "chp/dataset.hpp"
#include "chp/hulls.hpp"
#include "chp/reducer.hpp"

using chp::Point;

namespace {

std::vector<Point> widen(const int32_t* xy, uint64_t n) {
    std::vector<Point> pts(n);
    for (uint64_t i = 0; i < n; ++i) pts[i] = {xy[2 * i], xy[2 * i + 1]};
    return pts;
}

void narrow(const std::vector<Point>& v, int32_t* out) {
    for (size_t i = 0; i < v.size(); ++i) {
        out[2 * i] = static_cast<int32_t>(v[i].x);
        out[2 * i + 1] = static_cast<int32_t>(v[i].y);
    }
}

void L_pairs(const chp::reducer::ExtremalArray& arr, int32_t* out) {
    const int64_t w = arr.width();
    for (int64_t s = 0; s < w; ++s) {
        const auto& e = arr.entries[static_cast<size_t>(s)];
        out[2 * s] = e.valid ? static_cast<int32_t>(e.lo) : static_cast<int32_t>(w + 1);
        out[2 * s + 1] = e.valid ? static_cast<int32_t>(e.hi) : -1;
    }
}

}  // namespace

extern "C" {

// chp::dataset::generate({"uniform-box", n, p, seed}) narrowed to int32.
int ref_gen_uniform_box(uint64_t n, int64_t p, uint64_t seed, int32_t* xy) {
    chp::dataset::DatasetSpec spec;
    spec.source = "uniform-box";
    spec.n = static_cast<int64_t>(n);
    spec.p = p;
    spec.seed = seed;
    narrow(chp::dataset::generate(spec), xy);
    return 0;
}

// reduce -> L pairs (sentinel form), build_polyline -> chain, melkman -> hull.
// Any out pointer may be null.  Returns 0, -1 on std::invalid_argument from
// reduce, -2 when build_polyline throws (empty), -3 on other exceptions.
int ref_pipeline(const int32_t* xy, uint64_t n, int64_t width, int64_t q,
                 int32_t* L, int32_t* chain, int64_t* s, int32_t* hull,
                 int64_t* h, int64_t* valid_count) {
    const std::vector<Point> pts = widen(xy, n);
    std::optional<chp::reducer::ExtremalArray> opt;
    try {
        opt.emplace(q >= 0 ? chp::reducer::reduce(pts, width, q)
                           : chp::reducer::reduce(pts, width));
    } catch (const std::invalid_argument&) {
        return -1;
    }
    const chp::reducer::ExtremalArray& arr = *opt;
    if (L) L_pairs(arr, L);
    if (valid_count) *valid_count = arr.valid_count();
    chp::reducer::PolygonalChain c;
    try {
        c = chp::reducer::build_polyline(arr);
    } catch (const std::invalid_argument&) {
        if (s) *s = 0;
        return -2;
    }
    if (chain) narrow(c.vertices, chain);
    if (s) *s = static_cast<int64_t>(c.vertices.size());
    try {
        const chp::Hull hh = chp::hulls::melkman(c);
        if (hull) narrow(hh.vertices, hull);
        if (h) *h = static_cast<int64_t>(hh.vertices.size());
    } catch (...) {
        return -3;
    }
    return 0;
}

// serialize() text for reduce(pts, width[, q]); returns the text length or
// -1 on invalid input.  buf may be null (size query).
int64_t ref_serialize(const int32_t* xy, uint64_t n, int64_t width, int64_t q,
                      char* buf, int64_t cap) {
    const std::vector<Point> pts = widen(xy, n);
    try {
        const auto arr = q >= 0 ? chp::reducer::reduce(pts, width, q)
                                : chp::reducer::reduce(pts, width);
        std::ostringstream os;
        chp::reducer::serialize(arr, os);
        const std::string t = os.str();
        if (buf && static_cast<int64_t>(t.size()) <= cap) std::memcpy(buf, t.data(), t.size());
        return static_cast<int64_t>(t.size());
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// precondition(pts) -> bbox[4], major/minor offsets, chain, hull.
int ref_precondition(const int32_t* xy, uint64_t n, int64_t* bbox4,
                     int64_t* offsets2, int32_t* chain, int64_t* s,
                     int32_t* hull, int64_t* h) {
    const std::vector<Point> pts = widen(xy, n);
    try {
        const auto res = chp::reducer::precondition(pts);
        bbox4[0] = res.bbox.x_min;
        bbox4[1] = res.bbox.x_max;
        bbox4[2] = res.bbox.y_min;
        bbox4[3] = res.bbox.y_max;
        offsets2[0] = res.array.major_offset;
        offsets2[1] = res.array.minor_offset;
        if (chain) narrow(res.chain.vertices, chain);
        *s = static_cast<int64_t>(res.chain.vertices.size());
        const chp::Hull hh = chp::hulls::melkman(res.chain);
        if (hull) narrow(hh.vertices, hull);
        *h = static_cast<int64_t>(hh.vertices.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int64_t ref_melkman(const int32_t* chain, int64_t s, int32_t* hull) {
    chp::reducer::PolygonalChain c{widen(chain, static_cast<uint64_t>(s))};
    try {
        const chp::Hull hh = chp::hulls::melkman(c);
        narrow(hh.vertices, hull);
        return static_cast<int64_t>(hh.vertices.size());
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int64_t ref_graham(const int32_t* xy, int64_t n, int32_t* hull) {
    const auto pts = widen(xy, static_cast<uint64_t>(n));
    try {
        const chp::Hull hh = chp::hulls::graham_scan(pts);
        narrow(hh.vertices, hull);
        return static_cast<int64_t>(hh.vertices.size());
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// CPU baseline: time the reference's reduce + build_polyline over `n`
// int32 points split into `threads` contiguous chunks (one std::thread per
// chunk, each calling chp::reducer::reduce on its chunk; threads == 1 is the
// reference exactly as shipped).  Partial arrays are merged slot-wise and the
// merged survivors are passed through reduce once more to recover the exact
// ExtremalArray (idempotence, tests/test_reducer.cpp:113-127) before
// build_polyline.  The int32 -> chp::Point widening happens before the clock
// starts.  Returns seconds for `reps` repetitions (best), and s.
double ref_time_reduce_compact(const int32_t* xy, uint64_t n, int64_t width,
                               int64_t q, int threads, int reps, int64_t* s_out) {
    if (threads < 1) threads = 1;
    const std::vector<Point> pts = widen(xy, n);
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        std::optional<chp::reducer::ExtremalArray> arr;
        if (threads == 1) {
            arr.emplace(chp::reducer::reduce(pts, width, q));
        } else {
            std::vector<std::optional<chp::reducer::ExtremalArray>> part(
                static_cast<size_t>(threads));
            std::vector<std::thread> pool;
            for (int t = 0; t < threads; ++t) {
                const uint64_t b = n * static_cast<uint64_t>(t) / threads;
                const uint64_t e = n * static_cast<uint64_t>(t + 1) / threads;
                pool.emplace_back([&, t, b, e] {
                    part[static_cast<size_t>(t)].emplace(chp::reducer::reduce(
                        std::span<const Point>(pts.data() + b, e - b), width, q));
                });
            }
            for (auto& th : pool) th.join();
            std::vector<Point> survivors;
            for (const auto& a : part) {
                const auto v = a->valid_points();
                survivors.insert(survivors.end(), v.begin(), v.end());
            }
            arr.emplace(chp::reducer::reduce(survivors, width, q));
        }
        const auto chain = chp::reducer::build_polyline(*arr);
        const double dt =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (dt < best) best = dt;
        if (s_out) *s_out = static_cast<int64_t>(chain.vertices.size());
    }
    return best;
}

}  // extern "C"
