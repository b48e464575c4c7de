"""The Python mirror of the reference interface (paper_1505_00914_b200.reducer
/ .hulls / .kernels) on the device, against the reference's own KATs
(/root/reference/proj/tests/test_reducer.cpp, test_hulls.cpp,
test_kernels.cpp) and the oracle."""
import io

import numpy as np
import pytest

from _cases import mixed_case

pytestmark = pytest.mark.gpu

FIVE = [(1, 1), (1, 3), (1, 4), (2, 2), (2, 4), (3, 2), (3, 3), (3, 5), (4, 3), (5, 2), (5, 3), (2, 3), (3, 4)]


@pytest.fixture(scope="module")
def R(ctx):
    from paper_1505_00914_b200 import hulls, kernels, reducer

    return reducer, hulls, kernels


def valid_pairs(arr):
    return [(e.lo, e.hi) for e in arr.entries if e.valid]


def test_reduce_kats(R):
    reducer, _, _ = R
    arr = reducer.reduce(FIVE, 5)  # test_reducer.cpp:90-96
    assert valid_pairs(arr) == [(1, 4), (2, 4), (2, 5), (3, 3), (2, 3)]
    assert arr.valid_count() == 9
    one = reducer.reduce([(3, 7)], 5)  # :98-111
    assert [e.valid for e in one.entries] == [False, False, True, False, False]
    assert one.entries[2] == reducer.ColumnExtremes(7, 7, True)
    for bad, q in (((6, 1), None), ((0, 1), None), ((1, 0), None), ((1, 6), 5)):
        with pytest.raises(ValueError):
            reducer.reduce([bad], 5, q)
    with pytest.raises(ValueError):
        reducer.reduce([(1, 1)], 0)


def test_chain_serialize_kats(R):
    reducer, _, _ = R
    arr = reducer.reduce(FIVE, 5)
    assert reducer.build_polyline(arr).tolist() == [(1, 1), (1, 4), (2, 2), (2, 4), (3, 2), (3, 5), (4, 3), (5, 2),
                                                    (5, 3)]
    gaps = [(1, 1), (1, 4), (3, 2), (3, 5), (5, 2), (5, 3)]
    assert reducer.build_polyline(reducer.reduce(gaps, 5)).tolist() == gaps
    with pytest.raises(ValueError):
        reducer.build_polyline(reducer.reduce(np.empty((0, 2), np.int32), 5))
    buf = io.StringIO()
    text = reducer.serialize(reducer.reduce([(1, 4), (1, 1), (3, 9)], 4), buf)
    assert text == buf.getvalue() == "1 1 4\n2 5 -1\n3 9 9\n4 5 -1\n"


def test_precondition_kats(R, orc):
    reducer, hulls, _ = R
    res = reducer.precondition(FIVE)  # :225-244
    assert res.bbox == reducer.BoundingBox(1, 5, 1, 5)
    assert res.array.valid_count() == 9 and len(res.chain.vertices) == 9
    moved = [(x + 1000, y - 77) for x, y in FIVE]
    got = sorted(map(tuple, reducer.precondition(moved).array.valid_points().tolist()))
    assert got == [(1001, -76), (1001, -73), (1002, -75), (1002, -73), (1003, -75), (1003, -72), (1004, -74),
                   (1005, -75), (1005, -74)]
    assert reducer.precondition([(4, 4)]).chain.tolist() == [(4, 4)]
    with pytest.raises(ValueError):
        reducer.precondition([])
    # :268-284 auto_axis buckets along the short side, same hull
    rng = np.random.default_rng(67)
    flat = np.stack([rng.integers(1, 1001, 2000), rng.integers(1, 11, 2000)], axis=1)
    ax = reducer.precondition(flat, reducer.PreconditionOptions(auto_axis=True))
    assert ax.array.axis_swapped and ax.array.width() <= 10 and ax.array.valid_count() <= 20
    assert np.array_equal(orc.monotone_hull(ax.array.valid_points()), orc.monotone_hull(flat))
    # :296-304 second scan
    ss = reducer.precondition(FIVE, reducer.PreconditionOptions(second_scan=True))
    assert ss.array.axis_swapped
    assert np.array_equal(orc.monotone_hull(ss.array.valid_points()), orc.monotone_hull(FIVE))
    # :161-175 second_scan on the worked example
    sc = reducer.second_scan(reducer.reduce(FIVE, 5))
    assert sc.axis_swapped and valid_pairs(sc) == [(1, 1), (2, 5), (4, 5), (1, 2), (3, 3)]


def test_precondition_matches_reference_randomized(R, orc):
    reducer, hulls, _ = R
    rng = np.random.default_rng(71)
    for _ in range(60):
        pts = mixed_case(rng, int(rng.integers(1, 300)))
        res = reducer.precondition(pts)
        ref = orc.precondition(pts)
        assert (res.bbox.x_min, res.bbox.x_max, res.bbox.y_min, res.bbox.y_max) == ref["bbox"]
        assert np.array_equal(res.chain.vertices, ref["chain"])
        assert np.array_equal(hulls.melkman(res.chain).vertices, ref["hull"])


def test_hull_and_kernel_kats(R):
    reducer, hulls, kernels = R
    assert hulls.melkman(reducer.PolygonalChain(np.array([(0, 0), (4, 0), (2, 3)]))).tolist() == [(0, 0), (4, 0),
                                                                                                  (2, 3)]
    assert hulls.melkman(reducer.PolygonalChain(np.array([(3, 3)]))).tolist() == [(3, 3)]
    assert hulls.melkman(reducer.PolygonalChain(np.array([(0, 0), (2, 2), (5, 5)]))).tolist() == [(0, 0), (5, 5)]
    with pytest.raises(ValueError):
        hulls.melkman(reducer.PolygonalChain(np.empty((0, 2), np.int32)))
    m = kernels.min_max([(2, 3), (7, 1), (4, 9)])
    assert (m.x_min, m.x_max, m.y_min, m.y_max) == (2, 7, 1, 9)
    assert reducer.translate([(2, 3), (7, 1), (4, 9)], kernels.find_bounds([(2, 3), (7, 1), (4, 9)])).tolist() == \
        [[1, 3], [6, 1], [3, 9]]
    with pytest.raises(ValueError):
        kernels.min_max([])
    assert kernels.active_kernel() == "sm_100a"
