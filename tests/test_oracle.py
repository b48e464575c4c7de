"""The CPU oracle (oracle/chp_oracle.c) pinned to the reference: the golden
digests of SURVEY.md Appendix A (produced by the reference), the reference's
own KATs (tests/test_reducer.cpp, tests/test_hulls.cpp, acceptance.cpp), and
randomized equality with the reference library built from its own sources
(oracle/_ref/libchpref.so).  No GPU."""
import numpy as np
import pytest

from _cases import mixed_case, to_unit_box

FIVE = [(1, 1), (1, 3), (1, 4), (2, 2), (2, 4), (3, 2), (3, 3), (3, 5), (4, 3), (5, 2), (5, 3), (2, 3), (3, 4)]


def pairs(arr):
    return [(int(a), int(b)) for a, b, v in zip(arr["lo"], arr["hi"], arr["valid"]) if v]


def test_appendix_a_golden_digests(orc):
    xy = orc.uniform_box(1_000_000, 4096, 1)
    assert xy[:3].tolist() == [[549, 559], [1849, 87], [1438, 3733]]
    assert orc.fnv(xy) == "17239ebe0273b7d1"
    arr = orc.reduce(xy, 4096)
    assert orc.fnv(orc.L_pairs(arr)) == "b5b55891aaae7596"
    assert orc.fnv(orc.serialize(arr).encode()) == "75923f37d1030b80"
    chain = orc.build_polyline(arr)
    assert len(chain) == 8192 == orc.valid_count(arr)
    assert chain[:2].tolist() == [[1, 49], [1, 4071]] and chain[-1].tolist() == [4096, 4092]
    assert orc.fnv(chain) == "27d9354c9f73a66e"
    hull = orc.melkman(chain)
    assert hull.tolist() == [[1, 49], [2, 3], [15, 1], [4067, 1], [4093, 4], [4095, 7], [4096, 56], [4096, 4092],
                             [4093, 4096], [21, 4096], [3, 4091], [1, 4071]]
    assert np.array_equal(orc.monotone_hull(xy), hull)


def test_reducer_kats(orc):
    # test_reducer.cpp:90-96
    arr = orc.reduce(FIVE, 5)
    assert pairs(arr) == [(1, 4), (2, 4), (2, 5), (3, 3), (2, 3)]
    assert orc.valid_count(arr) == 9
    # :98-111
    one = orc.reduce([(3, 7)], 5)
    assert pairs(one) == [(7, 7)] and one["valid"].tolist() == [0, 0, 1, 0, 0]
    for bad, q in (((6, 1), None), ((0, 1), None), ((1, 0), None), ((1, 6), 5)):
        with pytest.raises(ValueError):
            orc.reduce([bad], 5, q)
    # :141-159
    assert pairs(orc.reduce([(2, 5)], 3)) == [(5, 5)]
    assert pairs(orc.reduce([(2, 5), (2, 8)], 3)) == [(5, 8)]
    assert pairs(orc.reduce([(2, 5), (2, 3)], 3)) == [(3, 5)]
    assert pairs(orc.reduce([(2, 3), (2, 8), (2, 9)], 3)) == [(3, 9)]
    assert pairs(orc.reduce([(2, 3), (2, 8), (2, 5)], 3)) == [(3, 8)]
    # :188-207
    assert orc.build_polyline(arr).tolist() == [[1, 1], [1, 4], [2, 2], [2, 4], [3, 2], [3, 5], [4, 3], [5, 2],
                                                [5, 3]]
    gaps = [(1, 1), (1, 4), (3, 2), (3, 5), (5, 2), (5, 3)]
    assert orc.build_polyline(orc.reduce(gaps, 5)).tolist() == [list(p) for p in gaps]
    with pytest.raises(ValueError):
        orc.build_polyline(orc.reduce(np.empty((0, 2), np.int32), 5))
    # :218-223
    assert orc.serialize(orc.reduce([(1, 4), (1, 1), (3, 9)], 4)) == "1 1 4\n2 5 -1\n3 9 9\n4 5 -1\n"


def test_hull_kats(orc):
    # test_hulls.cpp:104-128
    assert orc.melkman([(0, 0), (4, 0), (2, 3)]).tolist() == [[0, 0], [4, 0], [2, 3]]
    stair = [(i + d, i) for i in range(10) for d in (0, 1)]
    assert np.array_equal(orc.melkman(stair), orc.monotone_hull(stair))
    assert orc.melkman([(3, 3)]).tolist() == [[3, 3]]
    assert orc.melkman([(0, 0), (2, 2), (5, 5)]).tolist() == [[0, 0], [5, 5]]
    with pytest.raises(ValueError):
        orc.melkman(np.empty((0, 2), np.int32))
    # canonicalize (src/geometry.cpp:42-80)
    # clockwise, a collinear vertex, a duplicate -> CCW from the lex-min vertex
    assert orc.canonicalize([(0, 4), (4, 4), (4, 0), (2, 0), (2, 0), (0, 0)]).tolist() == [[0, 0], [4, 0], [4, 4],
                                                                                         [0, 4]]


def test_acceptance_c3_reduction_bound(orc):
    """acceptance.cpp:83-99: n=1e6, p=1000, seed 7 -> s = 2000 <= 2p."""
    xy = orc.uniform_box(1_000_000, 1000, 7)
    assert orc.valid_count(orc.reduce(xy, 1000)) == 2000


def test_melkman_equals_monotone_on_lemma1_chains(orc):
    rng = np.random.default_rng(11)
    for _ in range(300):
        pts, p = to_unit_box(mixed_case(rng, int(rng.integers(1, 300))))
        chain = orc.build_polyline(orc.reduce(pts, p))
        assert np.array_equal(orc.melkman(chain), orc.monotone_hull(pts))


def test_oracle_matches_reference_randomized(orc, ref):
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(1, 2000)) if trial % 40 else 100_000
        pts, p = to_unit_box(mixed_case(rng, n))
        q = None if trial % 3 else int(pts[:, 1].max())
        r = ref.pipeline(pts, p, q)
        arr = orc.reduce(pts, p, q)
        assert np.array_equal(r["L"], orc.L_pairs(arr))
        assert r["valid_count"] == orc.valid_count(arr)
        chain = orc.build_polyline(arr)
        assert np.array_equal(r["chain"], chain)
        assert np.array_equal(r["hull"], orc.melkman(chain))
        if trial % 20 == 0:
            assert ref.serialize(pts, p, q) == orc.serialize(arr)


def test_oracle_matches_reference_generator_and_validation(orc, ref):
    for n, p, seed in ((1000, 50, 3), (12345, 4096, 1), (1, 1, 9)):
        assert np.array_equal(orc.uniform_box(n, p, seed), ref.uniform_box(n, p, seed))
    with pytest.raises(ValueError):
        ref.pipeline([(6, 1)], 5)
    with pytest.raises(ValueError):
        orc.reduce([(6, 1)], 5)


def test_oracle_matches_reference_precondition(orc, ref):
    rng = np.random.default_rng(3)
    for _ in range(50):
        pts = mixed_case(rng, int(rng.integers(1, 500))).astype(np.int32)
        r = ref.precondition(pts)
        o = orc.precondition(pts)
        assert r["bbox"] == o["bbox"]
        assert r["major_offset"] == o["bbox"][0] - 1 and r["minor_offset"] == 0
        assert np.array_equal(r["chain"], o["chain"])
        assert np.array_equal(r["hull"], o["hull"])


def test_host_generator_lib_matches_product():
    """oracle/_build/libchpgen.so (what the CPU legs load instead of the
    product library) emits the product generator's bytes."""
    import oracle
    from paper_1505_00914_b200.device import generate_host

    for config, p in ((2, 65536), (3, 16384), (4, 1 << 20), (5, 256)):
        a = oracle.generate(config, config, p, 200_003, offset=987_654_321)
        b = generate_host(config, config, p, 200_003, offset=987_654_321)
        assert np.array_equal(a, b), config


def test_chunked_accumulator_matches_one_shot(orc):
    """SURVEY.md 8(c)'s chunked reduce (the full-size parity tests' oracle)
    equals one reduce() over the whole input."""
    import oracle

    for config, p in ((4, 1 << 20), (5, 256), (2, 4096)):
        xy = oracle.generate(config, config, p, 3_000_000)
        one = orc.reduce(xy, p, p)
        acc = orc.accumulator(p, p)
        for a in range(0, len(xy), 700_001):
            acc.add(xy[a:a + 700_001], threads=7)
        got = acc.finish()
        for k in ("lo", "hi", "valid", "occ"):
            v = one["valid"].astype(bool)
            if k in ("lo", "hi"):
                assert np.array_equal(got[k][v], one[k][v]), k
            else:
                assert np.array_equal(got[k], one[k]), k
    acc = orc.accumulator(10, 10)
    with pytest.raises(ValueError):
        acc.add(np.array([[1, 1], [11, 1]], np.int32))
