// chp/hulls.hpp -- drop-in for /root/reference/proj/include/chp/hulls.hpp:1-29.
// Upstream has four CPU hull algorithms plus a brute-force oracle, all
// returning the canonical Hull, so they agree by equality.  Here all of them
// return that same canonical hull computed on the device: the points are
// column-reduced (Algorithm 1 keeps every hull vertex, exactly) and the
// multi-level monotone chain of csrc/hull.cu runs on the lower and upper
// sequences (K4).  melkman() is the path's hull; the others keep their
// names and input checks (empty input, brute_force_hull's size bound).
// Device limit: the x extent of the input must be <= 2^29 columns
// (std::invalid_argument otherwise).
#pragma once

#include <cstddef>
#include <span>

#include "chp/geometry.hpp"
#include "chp/reducer.hpp"

namespace chp::hulls {

Hull graham_scan(std::span<const Point> points);

Hull quickhull(std::span<const Point> points);

Hull jarvis_march(std::span<const Point> points);

// Hull of a polygonal chain (a simple chain, as build_polyline emits; the
// device result is the exact hull of the chain's points for any chain).
Hull melkman(const reducer::PolygonalChain& chain);

// Refuses inputs larger than max_points, like upstream.
Hull brute_force_hull(std::span<const Point> points, std::size_t max_points = 500);

}  // namespace chp::hulls
