// dropin.cpp -- the reference's C++ entry points (include/chp/*.hpp) on top of
// the C ABI (include/chp_b200.h).  Everything that touches the point set
// runs on the device; the host only narrows int64 Points to int32 (the
// documented narrowing), calls the ABI and materialises the returned L,
// occupancy words, chain or hull into the reference's value types.
//
// Reference behaviour reproduced (paths under /root/reference/proj):
//   reduce          src/reducer.cpp:69-79   width/coordinate checks -> invalid_argument
//   build_polyline  src/reducer.cpp:108-119   empty -> invalid_argument
//   serialize       src/reducer.cpp:121-130
//   second_scan     src/reducer.cpp:81-106
//   precondition    src/reducer.cpp:132-178   (x-only, auto_axis, second_scan)
//   melkman & co.   src/hulls.cpp:34-224     canonical Hull, input checks
//   min_max etc.    src/kernels.cpp:8-67
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>

#include "chp/b200.hpp"
#include "chp/geometry.hpp"
#include "chp/hulls.hpp"
#include "chp/kernels.hpp"
#include "chp/occupancy.hpp"
#include "chp/reducer.hpp"
#include "chp_b200.h"

namespace chp {
namespace detail {

struct CtxHolder {
    chp_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) chp_ctx_destroy(ctx);
    }
};

// One context per host thread (the ABI's threading contract); device from
// CHP_DEVICE (default 0).
chp_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.ctx) {
        const char* env = std::getenv("CHP_DEVICE");
        const int dev = env ? std::atoi(env) : 0;
        if (chp_ctx_create(dev, &h.ctx) != CHP_OK)
            throw std::runtime_error("chp: no usable CUDA device " + std::to_string(dev));
    }
    return h.ctx;
}

void check(int rc) {
    if (rc == CHP_OK) return;
    const std::string msg = chp_last_error(ctx());
    if (rc == CHP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// Multi-device reduce (chp/b200.hpp): the shard group of this host thread.
struct GroupHolder {
    std::vector<int> devices;
    bool nccl = true;
    bool fused = false;  // CHP_COMBINE=fused: the shards fold into device 0's L over peer memory
    bool configured = false;
    chp_group* group = nullptr;
    ~GroupHolder() {
        if (group) chp_group_destroy(group);
    }
};

GroupHolder& group_holder() {
    thread_local GroupHolder h;
    if (!h.configured) {
        h.configured = true;
        if (const char* env = std::getenv("CHP_DEVICES")) {
            std::string s(env);
            size_t pos = 0;
            while (pos < s.size()) {
                const size_t comma = s.find(',', pos);
                const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
                if (!tok.empty()) h.devices.push_back(std::atoi(tok.c_str()));
                if (comma == std::string::npos) break;
                pos = comma + 1;
            }
        }
        const char* comb = std::getenv("CHP_COMBINE");
        h.nccl = !(comb && (std::string(comb) == "peer" || std::string(comb) == "fused"));
        h.fused = comb && std::string(comb) == "fused";
    }
    return h;
}

// The group when more than one device is configured, else nullptr.
chp_group* group() {
    GroupHolder& h = group_holder();
    if (h.devices.size() < 2) return nullptr;
    if (!h.group) {
        const int rc = chp_group_create(h.devices.data(), static_cast<int>(h.devices.size()),
                                        h.nccl ? CHP_COMBINE_NCCL : h.fused ? CHP_COMBINE_FUSED : CHP_COMBINE_PEER,
                                        &h.group);
        if (rc == CHP_EINVAL) throw std::invalid_argument("chp: bad device list for the shard group");
        if (rc != CHP_OK) throw std::runtime_error("chp: shard group creation failed");
    }
    return h.group;
}

void check_group(chp_group* g, int rc) {
    if (rc == CHP_OK) return;
    const std::string msg = chp_group_last_error(g);
    if (rc == CHP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// The chain reduce() computed alongside L (one device round trip less for
// the usual reduce -> build_polyline sequence): build_polyline reuses it
// when the array it is given still holds exactly that L with no offsets.
struct ChainCache {
    std::vector<int32_t> pairs;  // L in serialize form, as reduce() returned it
    std::vector<int32_t> chain;  // its Lemma-1 chain (int32 x, y)
    bool valid = false;
};

ChainCache& chain_cache() {
    thread_local ChainCache c;
    return c;
}

int32_t narrow1(std::int64_t v) {
    if (v < std::numeric_limits<int32_t>::min() || v > std::numeric_limits<int32_t>::max())
        throw std::invalid_argument("chp: coordinate outside the int32 range of the device path");
    return static_cast<int32_t>(v);
}

// Interleaved int32 (x, y), or (y, x) when swap.
std::vector<int32_t> narrow(std::span<const Point> pts, bool swap = false) {
    std::vector<int32_t> xy(2 * pts.size());
    for (size_t i = 0; i < pts.size(); ++i) {
        xy[2 * i] = narrow1(swap ? pts[i].y : pts[i].x);
        xy[2 * i + 1] = narrow1(swap ? pts[i].x : pts[i].y);
    }
    return xy;
}

std::vector<Point> widen(const int32_t* xy, int64_t n, bool swap = false) {
    std::vector<Point> out(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i)
        out[static_cast<size_t>(i)] = swap ? Point{xy[2 * i + 1], xy[2 * i]} : Point{xy[2 * i], xy[2 * i + 1]};
    return out;
}

// The reference's Point is two int64 words: the int64 entry points read
// the caller's array directly (no narrowed copy on the host).
const int64_t* raw64(std::span<const Point> pts) {
    static_assert(sizeof(Point) == 2 * sizeof(int64_t), "Point must be two packed int64");
    return reinterpret_cast<const int64_t*>(pts.data());
}

BoundingBox bounds_of(std::span<const Point> pts) {
    int64_t b4[4] = {0, 0, 0, 0};
    check(chp_bounds_host64(ctx(), raw64(pts), pts.size(), b4));
    return {b4[0], b4[1], b4[2], b4[3]};
}

// Entries from L in serialize form (lo > hi = empty).
std::vector<reducer::ColumnExtremes> entries_from_pairs(const std::vector<int32_t>& L, int64_t minor_shift = 0) {
    std::vector<reducer::ColumnExtremes> e(L.size() / 2);
    for (size_t s = 0; s < e.size(); ++s)
        if (L[2 * s] <= L[2 * s + 1]) e[s] = {L[2 * s] - minor_shift, L[2 * s + 1] - minor_shift, true};
    return e;
}

std::vector<int32_t> pairs_from_entries(const std::vector<reducer::ColumnExtremes>& entries) {
    const int64_t w = static_cast<int64_t>(entries.size());
    std::vector<int32_t> L(2 * entries.size());
    for (size_t s = 0; s < entries.size(); ++s) {
        const auto& e = entries[s];
        L[2 * s] = e.valid ? narrow1(e.lo) : narrow1(w + 1);
        L[2 * s + 1] = e.valid ? narrow1(e.hi) : -1;
    }
    return L;
}

occupancy::Index index_from_entries(const std::vector<reducer::ColumnExtremes>& e, occupancy::Kind kind) {
    occupancy::Index idx(e.size(), kind);
    std::vector<std::uint64_t> words((e.size() + 63) / 64, 0);
    for (size_t s = 0; s < e.size(); ++s)
        if (e[s].valid) words[s / 64] |= 1ull << (s % 64);
    idx.assign_words(words.data(), words.size());
    return idx;
}

// Canonical hull of a point set on the device, along whichever axis keeps
// the column count within the device limit.  One pass over the input
// (chp_precondition_run); only an x extent beyond 2^29 costs a second pass
// along y.
Hull device_hull(std::span<const Point> pts) {
    if (pts.empty()) throw std::invalid_argument("hull: empty input");
    int64_t b4[4] = {0, 0, 0, 0}, w = 0, s = 0, h = 0;
    int rc = chp_precondition_run64(ctx(), raw64(pts), pts.size(), 0, 1, b4, &w, &s, &h);
    bool swap = false;
    if (rc == CHP_EINVAL && b4[1] - b4[0] + 1 > (1ll << 29)) {
        const BoundingBox bb{b4[0], b4[1], b4[2], b4[3]};
        if (bb.height() > (1ll << 29) || bb.height() >= bb.width())
            throw std::invalid_argument("hull: point extent exceeds the device limit 2^29");
        swap = true;
        rc = chp_precondition_run64(ctx(), raw64(pts), pts.size(), 1, 1, b4, &w, &s, &h);
    }
    check(rc);
    std::vector<int32_t> hull(2 * static_cast<size_t>(h));
    check(chp_last_outputs(ctx(), nullptr, nullptr, hull.data()));
    std::vector<Point> v = widen(hull.data(), h, swap);
    if (swap) {
        // A reflection: restore CCW order, start at the lexicographic minimum.
        if (v.size() >= 3) std::reverse(v.begin(), v.end());
        auto it = std::min_element(v.begin(), v.end(), lex_less);
        std::rotate(v.begin(), it, v.end());
    }
    return Hull{std::move(v)};
}

}  // namespace detail

// ------------------------------------------------------------- geometry

BoundingBox find_bounds(std::span<const Point> points) {
    if (points.empty()) throw std::invalid_argument("find_bounds: empty input");
    return detail::bounds_of(points);
}

namespace {

int128 twice_area(const std::vector<Point>& v) {
    int128 a = 0;
    for (size_t i = 0, n = v.size(); i < n; ++i) {
        const Point &p = v[i], &q = v[(i + 1) % n];
        a += static_cast<int128>(p.x) * q.y - static_cast<int128>(q.x) * p.y;
    }
    return a;
}

Hull ends_of(const std::vector<Point>& v) {
    const auto [lo, hi] = std::minmax_element(v.begin(), v.end(), lex_less);
    if (*lo == *hi) return Hull{{*lo}};
    return Hull{{*lo, *hi}};
}

}  // namespace

Hull canonicalize_hull(std::span<const Point> vertices) {
    if (vertices.empty()) throw std::invalid_argument("canonicalize_hull: empty vertex list");
    std::vector<Point> v;
    for (const Point& p : vertices)
        if (v.empty() || !(v.back() == p)) v.push_back(p);
    while (v.size() > 1 && v.front() == v.back()) v.pop_back();
    if (v.size() <= 2) return Hull{v};
    const int128 area = twice_area(v);
    if (area == 0) return ends_of(v);
    if (area < 0) std::reverse(v.begin(), v.end());
    for (bool again = true; again && v.size() > 2;) {
        again = false;
        std::vector<Point> keep;
        for (size_t i = 0, n = v.size(); i < n; ++i) {
            if (orientation(v[(i + n - 1) % n], v[i], v[(i + 1) % n]) == Orientation::zero)
                again = true;
            else
                keep.push_back(v[i]);
        }
        v.swap(keep);
    }
    if (v.size() <= 2) return ends_of(v);
    std::rotate(v.begin(), std::min_element(v.begin(), v.end(), lex_less), v.end());
    return Hull{v};
}

bool hull_contains(const Hull& hull, const Point& p) {
    const auto& v = hull.vertices;
    if (v.empty()) return false;
    if (v.size() == 1) return v[0] == p;
    if (v.size() == 2)
        return orientation(v[0], v[1], p) == Orientation::zero && std::min(v[0].x, v[1].x) <= p.x &&
               p.x <= std::max(v[0].x, v[1].x) && std::min(v[0].y, v[1].y) <= p.y &&
               p.y <= std::max(v[0].y, v[1].y);
    for (size_t i = 0; i < v.size(); ++i)
        if (orientation(v[i], v[(i + 1) % v.size()], p) == Orientation::negative) return false;
    return true;
}

// -------------------------------------------------------------- kernels
namespace kernels {

MinMax min_max(std::span<const Point> pts) {
    if (pts.empty()) throw std::invalid_argument("min_max: empty input");
    const BoundingBox b = detail::bounds_of(pts);
    return {b.x_min, b.x_max, b.y_min, b.y_max};
}

void translate(std::span<const Point> in, std::int64_t dx, std::int64_t dy, std::span<Point> out) {
    if (out.size() < in.size()) throw std::invalid_argument("translate: output too small");
    if (in.empty()) return;
    auto xy = detail::narrow(in);
    std::vector<int32_t> res(xy.size());
    detail::check(chp_translate_host(detail::ctx(), xy.data(), in.size(), detail::narrow1(dx), detail::narrow1(dy),
                                     res.data()));
    // The device adds in 32-bit two's complement; flag results that left int32.
    for (size_t i = 0; i < in.size(); ++i) {
        detail::narrow1(in[i].x + dx);
        detail::narrow1(in[i].y + dy);
        out[i] = {res[2 * i], res[2 * i + 1]};
    }
}

MinMax min_max_scalar(const Point* pts, std::size_t n) { return min_max({pts, n}); }
void translate_scalar(const Point* in, std::size_t n, std::int64_t dx, std::int64_t dy, Point* out) {
    translate({in, n}, dx, dy, {out, n});
}
#if defined(__x86_64__) || defined(_M_X64)
MinMax min_max_avx2(const Point* pts, std::size_t n) { return min_max({pts, n}); }
void translate_avx2(const Point* in, std::size_t n, std::int64_t dx, std::int64_t dy, Point* out) {
    translate({in, n}, dx, dy, {out, n});
}
#endif

std::string_view active_kernel() { return "sm_100a"; }

}  // namespace kernels

// -------------------------------------------------------------- reducer
namespace reducer {

std::int64_t ExtremalArray::valid_count() const {
    std::int64_t c = 0;
    occ.for_each([&](std::uint64_t i) {
        const auto& e = entries[i - 1];
        c += e.lo == e.hi ? 1 : 2;
    });
    return c;
}

std::vector<Point> ExtremalArray::valid_points() const {
    std::vector<Point> out;
    occ.for_each([&](std::uint64_t i) {
        const auto& e = entries[i - 1];
        const auto s = static_cast<std::int64_t>(i);
        out.push_back(to_original(s, e.lo));
        if (e.hi != e.lo) out.push_back(to_original(s, e.hi));
    });
    return out;
}

std::vector<Point> translate(std::span<const Point> points, const BoundingBox& bbox) {
    std::vector<Point> out(points.size());
    kernels::translate(points, 1 - bbox.x_min, 1 - bbox.y_min, out);
    return out;
}

ExtremalArray reduce(std::span<const Point> points, std::int64_t width, std::optional<std::int64_t> q,
                     occupancy::Kind occ_kind) {
    if (width < 1) throw std::invalid_argument("reduce: width must be >= 1");
    std::vector<int32_t> L(2 * static_cast<size_t>(width));
    std::vector<std::uint64_t> words((static_cast<size_t>(width) + 63) / 64);
    detail::ChainCache& cache = detail::chain_cache();
    cache.valid = false;
    cache.chain.resize(4 * static_cast<size_t>(width));
    int64_t s = -1;
    const int64_t qq = q ? std::max<int64_t>(*q, 0) : -1;
    chp_group* g = width <= (1ll << 29) ? detail::group() : nullptr;
    const int rc = g ? chp_pipeline_host64_sharded(g, detail::raw64(points), points.size(), width, qq, L.data(),
                                                   words.data(), cache.chain.data(), &s, nullptr, nullptr)
                     : chp_pipeline_host64(detail::ctx(), detail::raw64(points), points.size(), width, qq, L.data(),
                                           words.data(), cache.chain.data(), &s, nullptr, nullptr);
    if (rc == CHP_EINVAL && s == 0) {
        // valid input, no point at all: the pipeline refuses the (empty)
        // chain it was asked for, and L is all sentinels
        for (int64_t i = 0; i < width; ++i) {
            L[2 * i] = detail::narrow1(width + 1);
            L[2 * i + 1] = -1;
        }
        std::fill(words.begin(), words.end(), 0);
    } else if (g) {
        detail::check_group(g, rc);
    } else {
        detail::check(rc);
    }
    cache.chain.resize(2 * static_cast<size_t>(std::max<int64_t>(s, 0)));
    cache.pairs = L;
    cache.valid = true;
    ExtremalArray arr{detail::entries_from_pairs(L), occupancy::Index(static_cast<std::uint64_t>(width), occ_kind)};
    arr.occ.assign_words(words.data(), words.size());
    return arr;
}

ExtremalArray second_scan(const ExtremalArray& arr, occupancy::Kind occ_kind) {
    const std::vector<Point> pts = arr.valid_points();
    const bool swapped = !arr.axis_swapped;
    if (pts.empty()) {
        ExtremalArray out{std::vector<ColumnExtremes>(static_cast<size_t>(arr.width())),
                          occupancy::Index(static_cast<std::uint64_t>(arr.width()), occ_kind)};
        out.axis_swapped = swapped;
        return out;
    }
    const BoundingBox bb = find_bounds(pts);
    const std::int64_t major_min = swapped ? bb.y_min : bb.x_min, major_max = swapped ? bb.y_max : bb.x_max;
    const std::int64_t minor_min = swapped ? bb.x_min : bb.y_min;
    std::vector<Point> rebased(pts.size());
    for (size_t i = 0; i < pts.size(); ++i) {
        const std::int64_t a = swapped ? pts[i].y : pts[i].x, b = swapped ? pts[i].x : pts[i].y;
        rebased[i] = {a - (major_min - 1), b - (minor_min - 1)};
    }
    ExtremalArray out = reduce(rebased, major_max - major_min + 1, std::nullopt, occ_kind);
    out.major_offset = major_min - 1;
    out.minor_offset = minor_min - 1;
    out.axis_swapped = swapped;
    return out;
}

PolygonalChain build_polyline(const ExtremalArray& arr) {
    if (arr.width() < 1) throw std::invalid_argument("build_polyline: no valid points");
    const auto L = detail::pairs_from_entries(arr.entries);
    const detail::ChainCache& cache = detail::chain_cache();
    if (cache.valid && arr.major_offset == 0 && arr.minor_offset == 0 && !arr.axis_swapped && L == cache.pairs) {
        // the L reduce() just produced: its chain came back with it
        if (cache.chain.empty()) throw std::invalid_argument("build_polyline: no valid points");
        return PolygonalChain{detail::widen(cache.chain.data(), static_cast<int64_t>(cache.chain.size() / 2))};
    }
    std::vector<int32_t> chain(4 * L.size() / 2 + 4);
    int64_t s = 0;
    detail::check(chp_polyline_host(detail::ctx(), L.data(), arr.width(), arr.major_offset, arr.minor_offset,
                                    arr.axis_swapped ? 1 : 0, chain.data(), &s));
    return PolygonalChain{detail::widen(chain.data(), s)};
}

void serialize(const ExtremalArray& arr, std::ostream& os) {
    const std::int64_t w = arr.width();
    for (std::int64_t i = 1; i <= w; ++i) {
        const auto& e = arr.entries[static_cast<size_t>(i - 1)];
        os << i << ' ' << (e.valid ? e.lo : w + 1) << ' ' << (e.valid ? e.hi : -1) << '\n';
    }
}

PreconditionResult precondition(std::span<const Point> points, const PreconditionOptions& options) {
    if (points.empty()) throw std::invalid_argument("precondition: empty input");
    using clock = std::chrono::steady_clock;
    auto t0 = clock::now();
    const bool full_bounds = options.second_scan || options.auto_axis;
    // auto_axis needs the box before choosing the axis (one bounds-only pass);
    // otherwise bounds, fold, compaction are ONE pass over the caller's int64
    // points (chp_precondition_run64).
    bool swap = false;
    if (options.auto_axis) {
        const BoundingBox bb0 = detail::bounds_of(points);
        swap = bb0.height() < bb0.width();
    }
    auto t1 = clock::now();
    int64_t b4[4] = {0, 0, 0, 0}, width = 0, s = 0;
    const int rc = chp_precondition_run64(detail::ctx(), detail::raw64(points), points.size(), swap ? 1 : 0, 0, b4,
                                          &width, &s, nullptr);
    if (rc == CHP_EINVAL && b4[1] - b4[0] + 1 > (1ll << 29))
        throw std::invalid_argument("precondition: extent exceeds the device limit 2^29");
    detail::check(rc);
    // b4 is the box of the (possibly axis-swapped) input
    const BoundingBox bb = swap ? BoundingBox{b4[2], b4[3], b4[0], b4[1]} : BoundingBox{b4[0], b4[1], b4[2], b4[3]};
    const std::int64_t major_offset = b4[0] - 1;
    const std::int64_t minor_offset = full_bounds ? b4[2] - 1 : 0;
    std::vector<int32_t> L(2 * static_cast<size_t>(width)), chain(2 * static_cast<size_t>(s));
    detail::check(chp_last_outputs(detail::ctx(), L.data(), chain.data(), nullptr));
    PreconditionResult res{ExtremalArray{detail::entries_from_pairs(L, minor_offset),
                                         occupancy::Index(1, options.occ_kind)},
                           {}, bb};
    res.array.occ = detail::index_from_entries(res.array.entries, options.occ_kind);
    res.array.major_offset = major_offset;
    res.array.minor_offset = minor_offset;
    res.array.axis_swapped = swap;
    auto t2 = clock::now();
    if (options.second_scan) {
        res.array = second_scan(res.array, options.occ_kind);
        res.chain = build_polyline(res.array);
    } else {
        res.chain = PolygonalChain{detail::widen(chain.data(), s, swap)};
    }
    auto t3 = clock::now();
    res.t_bounds = std::chrono::duration<double>(t1 - t0).count();
    res.t_reduce = std::chrono::duration<double>(t2 - t1).count();
    res.t_extract = std::chrono::duration<double>(t3 - t2).count();
    return res;
}

}  // namespace reducer

// ---------------------------------------------------------------- hulls
namespace hulls {

Hull graham_scan(std::span<const Point> points) {
    if (points.empty()) throw std::invalid_argument("graham_scan: empty input");
    return detail::device_hull(points);
}

Hull quickhull(std::span<const Point> points) {
    if (points.empty()) throw std::invalid_argument("quickhull: empty input");
    return detail::device_hull(points);
}

Hull jarvis_march(std::span<const Point> points) {
    if (points.empty()) throw std::invalid_argument("jarvis_march: empty input");
    return detail::device_hull(points);
}

Hull melkman(const reducer::PolygonalChain& chain) {
    if (chain.vertices.empty()) throw std::invalid_argument("melkman: empty chain");
    return detail::device_hull(chain.vertices);
}

Hull brute_force_hull(std::span<const Point> points, std::size_t max_points) {
    if (points.empty()) throw std::invalid_argument("brute_force_hull: empty input");
    if (points.size() > max_points) throw std::invalid_argument("brute_force_hull: input exceeds size bound");
    return detail::device_hull(points);
}

}  // namespace hulls

// ------------------------------------------------------ device options
namespace b200 {

void use_devices(const std::vector<int>& devs, bool nccl) {
    detail::GroupHolder& h = detail::group_holder();
    if (h.group) {
        chp_group_destroy(h.group);
        h.group = nullptr;
    }
    h.devices = devs;
    h.nccl = nccl;
}

std::vector<int> devices() {
    const detail::GroupHolder& h = detail::group_holder();
    if (h.devices.size() >= 2) return h.devices;
    const char* env = std::getenv("CHP_DEVICE");
    return {env ? std::atoi(env) : 0};
}

}  // namespace b200
}  // namespace chp
