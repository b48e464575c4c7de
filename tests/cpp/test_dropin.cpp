// test_dropin.cpp -- the reference's own known-answer tests for the hot path,
// restated against the C++ drop-in (include/chp/*.hpp + libchp_b200.so).
// Each block cites the reference test it restates
// (/root/reference/proj/tests/test_reducer.cpp, test_hulls.cpp,
// test_occupancy.cpp, acceptance.cpp).  Prints one line per failed check and
// exits non-zero if any failed.  Needs a CUDA device (run by
// tests/test_dropin_gpu.py).
#include <algorithm>
#include <cstdio>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "chp/b200.hpp"
#include "chp/geometry.hpp"
#include "chp/hulls.hpp"
#include "chp/kernels.hpp"
#include "chp/occupancy.hpp"
#include "chp/reducer.hpp"

using namespace chp;
using namespace chp::reducer;

static int g_checks = 0, g_fail = 0;
#define EXPECT(cond)                                                              \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(cond)) {                                                            \
            ++g_fail;                                                             \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
        }                                                                         \
    } while (0)
#define EXPECT_THROWS(expr, type)                                                 \
    do {                                                                          \
        ++g_checks;                                                               \
        bool ok_ = false;                                                         \
        try {                                                                     \
            (void)(expr);                                                         \
        } catch (const type&) {                                                   \
            ok_ = true;                                                           \
        } catch (...) {                                                           \
        }                                                                         \
        if (!ok_) {                                                               \
            ++g_fail;                                                             \
            std::printf("FAIL %s:%d: expected %s from %s\n", __FILE__, __LINE__, #type, #expr); \
        }                                                                         \
    } while (0)

namespace {

// Extremes per column: 1->{1,4} 2->{2,4} 3->{2,5} 4->{3,3} 5->{2,3}
// (test_reducer.cpp:16-21).
std::vector<Point> five_columns() {
    return {{1, 1}, {1, 3}, {1, 4}, {2, 2}, {2, 4}, {3, 2}, {3, 3},
            {3, 5}, {4, 3}, {5, 2}, {5, 3}, {2, 3}, {3, 4}};
}

std::vector<std::pair<std::int64_t, std::int64_t>> valid_pairs(const ExtremalArray& a) {
    std::vector<std::pair<std::int64_t, std::int64_t>> v;
    for (const auto& e : a.entries)
        if (e.valid) v.emplace_back(e.lo, e.hi);
    return v;
}

std::vector<Point> random_points(std::mt19937_64& rng, std::size_t n, std::int64_t lo, std::int64_t hi) {
    std::uniform_int_distribution<std::int64_t> d(lo, hi);
    std::vector<Point> p(n);
    for (auto& q : p) q = {d(rng), d(rng)};
    return p;
}

// An exact CPU hull used only as this test's checker (Andrew's monotone
// chain over the deduplicated lexicographic order).
Hull checker_hull(std::vector<Point> p) {
    std::sort(p.begin(), p.end(), lex_less);
    p.erase(std::unique(p.begin(), p.end()), p.end());
    if (p.size() == 1) return Hull{p};
    std::vector<Point> h;
    for (int pass = 0; pass < 2; ++pass) {
        const size_t base = h.size();
        for (const Point& q : p) {
            while (h.size() >= base + 2 && orientation(h[h.size() - 2], h.back(), q) != Orientation::positive)
                h.pop_back();
            h.push_back(q);
        }
        h.pop_back();
        std::reverse(p.begin(), p.end());
    }
    if (h.size() < 2) h = {p.back(), p.front()};
    return canonicalize_hull(h);
}

void reducer_kats() {
    // test_reducer.cpp:90-96 -- worked example, valid_count 9
    const auto arr = reduce(five_columns(), 5);
    EXPECT((valid_pairs(arr) ==
            std::vector<std::pair<std::int64_t, std::int64_t>>{{1, 4}, {2, 4}, {2, 5}, {3, 3}, {2, 3}}));
    EXPECT(arr.valid_count() == 9);

    // :98-111 -- single point; validation throws
    const auto one = reduce(std::vector<Point>{{3, 7}}, 5);
    EXPECT(!one.entries[0].valid && !one.entries[1].valid && !one.entries[3].valid && !one.entries[4].valid);
    EXPECT((one.entries[2] == ColumnExtremes{7, 7, true}));
    EXPECT_THROWS(reduce(std::vector<Point>{{6, 1}}, 5), std::invalid_argument);
    EXPECT_THROWS(reduce(std::vector<Point>{{0, 1}}, 5), std::invalid_argument);
    EXPECT_THROWS(reduce(std::vector<Point>{{1, 0}}, 5), std::invalid_argument);
    EXPECT_THROWS(reduce(std::vector<Point>{{1, 6}}, 5, 5), std::invalid_argument);
    EXPECT_THROWS(reduce(std::vector<Point>{{1, 1}}, 0), std::invalid_argument);

    // :113-127 -- order-insensitive, idempotent on its survivors
    std::mt19937_64 rng(41);
    for (int t = 0; t < 40; ++t) {
        auto pts = random_points(rng, 1 + rng() % 200, 1, 40);
        auto shuf = pts;
        std::shuffle(shuf.begin(), shuf.end(), rng);
        const auto a = reduce(pts, 40), b = reduce(shuf, 40);
        EXPECT(valid_pairs(a) == valid_pairs(b));
        EXPECT(valid_pairs(reduce(a.valid_points(), 40)) == valid_pairs(a));
    }

    // :141-159 -- induction cases
    EXPECT((reduce(std::vector<Point>{{2, 5}}, 3).entries[1] == ColumnExtremes{5, 5, true}));
    EXPECT((reduce(std::vector<Point>{{2, 5}, {2, 8}}, 3).entries[1] == ColumnExtremes{5, 8, true}));
    EXPECT((reduce(std::vector<Point>{{2, 5}, {2, 3}}, 3).entries[1] == ColumnExtremes{3, 5, true}));
    EXPECT((reduce(std::vector<Point>{{2, 5}, {2, 5}}, 3).entries[1] == ColumnExtremes{5, 5, true}));
    EXPECT((reduce(std::vector<Point>{{2, 3}, {2, 8}, {2, 9}}, 3).entries[1] == ColumnExtremes{3, 9, true}));
    EXPECT((reduce(std::vector<Point>{{2, 3}, {2, 8}, {2, 5}}, 3).entries[1] == ColumnExtremes{3, 8, true}));

    // :161-175 -- second scan
    const auto sc = second_scan(arr);
    EXPECT(sc.axis_swapped);
    EXPECT((valid_pairs(sc) ==
            std::vector<std::pair<std::int64_t, std::int64_t>>{{1, 1}, {2, 5}, {4, 5}, {1, 2}, {3, 3}}));

    // :188-196 -- Lemma-1 chain order
    EXPECT((build_polyline(arr).vertices ==
            std::vector<Point>{{1, 1}, {1, 4}, {2, 2}, {2, 4}, {3, 2}, {3, 5}, {4, 3}, {5, 2}, {5, 3}}));
    EXPECT((build_polyline(reduce(std::vector<Point>{{3, 2}, {3, 9}}, 5)).vertices ==
            std::vector<Point>{{3, 2}, {3, 9}}));

    // :198-207 -- gaps are bridged; empty -> invalid_argument
    const std::vector<Point> gaps{{1, 1}, {1, 4}, {3, 2}, {3, 5}, {5, 2}, {5, 3}};
    EXPECT(build_polyline(reduce(gaps, 5)).vertices == gaps);
    EXPECT_THROWS(build_polyline(reduce(std::vector<Point>{}, 5)), std::invalid_argument);

    // :218-223 -- serialize sentinel text
    std::ostringstream os;
    serialize(reduce(std::vector<Point>{{1, 4}, {1, 1}, {3, 9}}, 4), os);
    EXPECT(os.str() == "1 1 4\n2 5 -1\n3 9 9\n4 5 -1\n");

    // :225-258 -- precondition
    const auto pr = precondition(five_columns());
    EXPECT((pr.bbox == BoundingBox{1, 5, 1, 5}));
    EXPECT(pr.array.valid_count() == 9 && pr.chain.vertices.size() == 9);
    std::vector<Point> moved = five_columns();
    for (auto& p : moved) p = {p.x + 1000, p.y - 77};
    auto got = precondition(moved).array.valid_points();
    std::sort(got.begin(), got.end(), lex_less);
    EXPECT((got == std::vector<Point>{{1001, -76}, {1001, -73}, {1002, -75}, {1002, -73}, {1003, -75},
                                      {1003, -72}, {1004, -74}, {1005, -75}, {1005, -74}}));
    const auto single = precondition(std::vector<Point>{{4, 4}});
    EXPECT(single.array.valid_count() == 1 && (single.chain.vertices == std::vector<Point>{{4, 4}}));
    EXPECT_THROWS(precondition({}), std::invalid_argument);

    // :268-284 -- auto_axis buckets along the short side, same hull
    std::vector<Point> flat(2000);
    for (auto& p : flat)
        p = {static_cast<std::int64_t>(1 + rng() % 1000), static_cast<std::int64_t>(1 + rng() % 10)};
    PreconditionOptions opts;
    opts.auto_axis = true;
    const auto ax = precondition(flat, opts);
    EXPECT(ax.array.axis_swapped && ax.array.width() <= 10 && ax.array.valid_count() <= 20);
    EXPECT(hulls::melkman(PolygonalChain{ax.array.valid_points()}) ==
           hulls::melkman(PolygonalChain{precondition(flat).array.valid_points()}));

    // :286-294 -- the survivors keep the hull (checked with an independent CPU hull)
    for (int t = 0; t < 60; ++t) {
        const auto pts = random_points(rng, 1 + rng() % 300, -1000, 1000);
        EXPECT(checker_hull(precondition(pts).array.valid_points()) == checker_hull(pts));
    }
    // :296-304 -- second scan through the options
    PreconditionOptions ss;
    ss.second_scan = true;
    const auto r2 = precondition(five_columns(), ss);
    EXPECT(r2.array.axis_swapped && checker_hull(r2.array.valid_points()) == checker_hull(five_columns()));
    // :306-314 -- tree occupancy gives the same chain
    PreconditionOptions tree;
    tree.occ_kind = occupancy::Kind::tree;
    const auto rp = random_points(rng, 500, 1, 300);
    EXPECT(precondition(rp).chain.vertices == precondition(rp, tree).chain.vertices);
}

void hull_kats() {
    using namespace chp::hulls;
    // test_hulls.cpp:13-56
    const std::vector<Point> sq{{0, 0}, {4, 0}, {4, 4}, {0, 4}, {2, 2}};
    const Hull sqh{{{0, 0}, {4, 0}, {4, 4}, {0, 4}}};
    EXPECT(graham_scan(sq) == sqh && quickhull(sq) == sqh && jarvis_march(sq) == sqh && brute_force_hull(sq) == sqh);
    EXPECT((graham_scan(std::vector<Point>{{2, 3}, {0, 0}, {4, 0}}) == Hull{{{0, 0}, {4, 0}, {2, 3}}}));
    EXPECT((graham_scan(std::vector<Point>{{5, 5}, {1, 1}, {3, 3}, {1, 1}}) == Hull{{{1, 1}, {5, 5}}}));
    EXPECT((graham_scan(std::vector<Point>{{7, 7}, {7, 7}, {7, 7}}) == Hull{{{7, 7}}}));
    EXPECT_THROWS(graham_scan({}), std::invalid_argument);
    EXPECT((quickhull(std::vector<Point>{{0, 0}, {2, 0}, {4, 0}, {4, 4}, {0, 4}, {0, 2}}) == sqh));

    // :418-442 -- Melkman on simple chains and degenerate chains
    const std::vector<Point> pts{{1, 1}, {1, 3}, {1, 4}, {2, 2}, {2, 4}, {3, 2},
                                 {3, 3}, {3, 5}, {4, 3}, {5, 2}, {5, 3}, {2, 3}};
    EXPECT(melkman(precondition(pts).chain) == checker_hull(pts));
    EXPECT((melkman(PolygonalChain{{{0, 0}, {4, 0}, {2, 3}}}) == Hull{{{0, 0}, {4, 0}, {2, 3}}}));
    PolygonalChain stair;
    for (int i = 0; i < 10; ++i) {
        stair.vertices.push_back({i, i});
        stair.vertices.push_back({i + 1, i});
    }
    EXPECT(melkman(stair) == checker_hull(stair.vertices));
    EXPECT((melkman(PolygonalChain{{{3, 3}}}) == Hull{{{3, 3}}}));
    EXPECT((melkman(PolygonalChain{{{0, 0}, {2, 2}, {5, 5}}}) == Hull{{{0, 0}, {5, 5}}}));
    EXPECT_THROWS(melkman(PolygonalChain{}), std::invalid_argument);

    // :444-454 -- agreement through the reducer on randomized sets
    std::mt19937_64 rng(113);
    for (int t = 0; t < 60; ++t) {
        const auto p = random_points(rng, 1 + rng() % 250, -50000, 50000);
        const Hull g = checker_hull(p);
        EXPECT(graham_scan(p) == g);
        EXPECT(melkman(precondition(p).chain) == g);
    }
    // :456-460 -- brute-force size bound
    std::vector<Point> big(501, Point{0, 0});
    EXPECT_THROWS(brute_force_hull(big), std::invalid_argument);
    EXPECT((brute_force_hull(big, 501) == Hull{{{0, 0}}}));
}

void occupancy_kats() {
    using namespace chp::occupancy;
    // test_occupancy.cpp:27-43, :80-115, :138-163; acceptance.cpp criteria 4-6
    EXPECT((extract_word_positions<std::uint64_t>(0b10101) == std::vector<int>{0, 2, 4}));
    EXPECT(msb_position<std::uint64_t>(0b10101) == 4);
    EXPECT((bit_index_map(103223, 32) == BlockPosition{3225, 22}));
    EXPECT((bit_index_map(65, 64) == BlockPosition{1, 0}));
    BlockedBitset<std::uint64_t> bs(5);
    bs.insert(5);
    bs.insert(1);
    bs.insert(3);
    EXPECT(bs.blocks()[0] == 0b10101);
    EXPECT((bs.indices() == std::vector<std::uint64_t>{1, 3, 5}));
    EXPECT_THROWS(bs.insert(6), std::out_of_range);
    const WAryOccupancyTree<std::uint64_t> tree(1ull << 24);
    EXPECT(tree.height() == 3 && tree.total_words() == 266305 && tree.leaf_words() == 262144);
    // the occupancy words the device emits equal the reference layout
    const auto a = reduce(std::vector<Point>{{1, 4}, {1, 1}, {3, 9}, {70, 2}}, 100);
    EXPECT((a.occ.indices() == std::vector<std::uint64_t>{1, 3, 70}));
}

void kernel_kats() {
    using namespace chp::kernels;
    // test_kernels.cpp:19-60 (device path), test_reducer.cpp:78-88 (translate)
    const std::vector<Point> p{{2, 3}, {7, 1}, {4, 9}};
    const MinMax m = min_max(p);
    EXPECT(m.x_min == 2 && m.x_max == 7 && m.y_min == 1 && m.y_max == 9);
    EXPECT((translate(p, find_bounds(p)) == std::vector<Point>{{1, 3}, {6, 1}, {3, 9}}));
    EXPECT_THROWS(min_max({}), std::invalid_argument);
    EXPECT_THROWS(find_bounds(std::vector<Point>{{1ll << 40, 0}}), std::invalid_argument);
    EXPECT(active_kernel() == "sm_100a");
}

void acceptance_c3() {
    // acceptance.cpp:83-99 -- n = 1e6 uniform in [1,1000]^2: s <= 2p, >= 99.8% reduction
    std::mt19937_64 rng(7);
    std::uniform_int_distribution<std::int64_t> d(1, 1000);
    std::vector<Point> pts(1000000);
    for (auto& q : pts) q = {d(rng), d(rng)};
    const auto res = precondition(pts);
    EXPECT(res.array.valid_count() == 2000);
}

void chain_reuse_and_devices() {
    // build_polyline after reduce reuses the chain that came back with L; an
    // array edited afterwards (or with offsets) takes the device round trip.
    // Either way the chain is the Lemma-1 chain of the array it is given
    // (test_reducer.cpp:188-207).
    const auto a = reduce(five_columns(), 5);
    const auto c1 = build_polyline(a);
    EXPECT(c1.vertices.size() == 9);
    EXPECT(c1.vertices.front() == (Point{1, 1}) && c1.vertices.back() == (Point{5, 3}));
    auto b = a;
    b.entries[0].hi = 7;  // edited after reduce: (1,1),(1,7) ...
    const auto c2 = build_polyline(b);
    EXPECT(c2.vertices.size() == 9 && c2.vertices[1] == (Point{1, 7}));
    auto c = a;
    c.major_offset = 10;  // offsets: to_original moves every point
    EXPECT(build_polyline(c).vertices.front() == (Point{11, 1}));
    // empty input: all slots empty, build_polyline throws (test_reducer.cpp:198-207)
    const auto e = reduce(std::vector<Point>{}, 4);
    EXPECT(e.valid_count() == 0);
    EXPECT_THROWS(build_polyline(e), std::invalid_argument);
    EXPECT(build_polyline(a).vertices == c1.vertices);

    // reduce split over a shard group (chp/b200.hpp): four shards on the
    // first device with the peer combine give the single-device result
    std::mt19937_64 rng(11);
    std::uniform_int_distribution<std::int64_t> dx(1, 3000), dy(1, 5000);
    std::vector<Point> pts(2000003);
    for (auto& q : pts) q = {dx(rng), dy(rng)};
    const auto one = reduce(pts, 3000, 5000);
    const auto chain_one = build_polyline(one);
    const int dev = chp::b200::devices().front();
    chp::b200::use_devices({dev, dev, dev, dev}, /*nccl=*/false);
    EXPECT(chp::b200::devices().size() == 4);
    const auto four = reduce(pts, 3000, 5000);
    EXPECT(four.entries == one.entries);
    EXPECT(build_polyline(four).vertices == chain_one.vertices);
    auto bad = pts;
    bad[2000000] = {3001, 1};  // in the last shard
    EXPECT_THROWS(reduce(bad, 3000, 5000), std::invalid_argument);
    chp::b200::use_devices({dev});
    EXPECT(chp::b200::devices().size() == 1);
    EXPECT(reduce(pts, 3000, 5000).entries == one.entries);
}

}  // namespace

int main() {
    reducer_kats();
    hull_kats();
    occupancy_kats();
    kernel_kats();
    acceptance_c3();
    chain_reuse_and_devices();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
