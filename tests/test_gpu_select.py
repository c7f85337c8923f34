"""GPU parity: hot-set selection (K4-K6) and the reorder ops. Bit-exact
(integer outputs compared for equality)."""
import numpy as np
import pytest

import oracle
from tests.helpers import random_graph, random_permutation

pytestmark = pytest.mark.gpu


def test_known_answers(tg, ctx):
    assert list(tg.score_ordering([0.1, 0.4, 0.2, 0.3])) == [1, 3, 2, 0]  # test_scoring.cpp:145-149
    assert list(tg.score_ordering([7.0, 7.0, 7.0])) == [0, 1, 2]
    assert list(tg.score_ordering([5.0, 5.0, 1.0])) == [0, 1, 2]
    assert list(tg.permutation_from_scores([0.1, 0.4, 0.2, 0.3]).new_id_of) == [3, 0, 2, 1]
    assert list(tg.permutation_from_scores([9.0, 8.0, 7.0]).new_id_of) == [0, 1, 2]
    assert list(tg.permutation_from_scores([1.0, 1.0, 1.0]).new_id_of) == [0, 1, 2]
    s = [0.3, 0.9, 0.9, 0.1, 0.5]
    order, perm = tg.score_ordering(s), tg.permutation_from_scores(s).new_id_of
    assert all(perm[order[r]] == r for r in range(5))
    assert list(tg.invert([3, 0, 2, 1]).new_id_of) == [1, 3, 2, 0]
    assert tg.score_ordering([]).size == 0


def test_signed_zero_and_rejects(tg, ctx):
    assert list(tg.score_ordering([0.0, -0.0, 0.0, 1e-300, -0.0])) == [3, 0, 1, 2, 4]
    for bad, idx in (([0.1, float("nan")], 1), ([float("inf")], 0), ([1.0, 2.0, -1e-300], 2),
                     ([0.0] * 5000 + [float("-inf")] + [float("nan")], 5000)):
        with pytest.raises(tg.DomainError, match=f"score {idx} is not finite"):
            tg.score_ordering(bad)


@pytest.mark.parametrize("n", [1, 31, 4095, 4096, 4097, 100_003, 1_300_000])
def test_random_scores_with_ties(tg, ctx, n):
    rng = np.random.default_rng(n)
    # heavy ties + wide exponent range + exact zeros
    s = np.where(rng.random(n) < 0.3, np.floor(rng.random(n) * 50) / 64,
                 rng.random(n) * 10.0 ** rng.integers(-300, 3, n))
    s[rng.random(n) < 0.05] = 0.0
    want = oracle.port().score_ordering(s)
    assert np.array_equal(tg.score_ordering(s), want)
    p = tg.permutation_from_scores(s).new_id_of
    assert np.array_equal(p, oracle.port().permutation_from_scores(s))


@pytest.mark.parametrize("n", [2, 4096, 100_003, 1_300_000])
def test_lowest_score_ties_compacted(tg, ctx, n):
    """>= 1/8 of the scores equal the minimum (reverse PageRank: every node
    without out-edges scores exactly the teleport term): those ids leave the
    radix sort and go last in id order; -0.0 and +0.0 minima tie."""
    rng = np.random.default_rng(n + 7)
    base = 0.15 / max(n, 1)
    s = base + rng.random(n) * 10.0 ** rng.integers(-12, -3, n)
    s[rng.random(n) < 0.6] = base
    s[0] = base
    z = np.where(rng.random(n) < 0.3, np.where(rng.random(n) < 0.5, -0.0, 0.0), s)
    port = oracle.port()
    for case in (s, z):
        assert np.array_equal(tg.score_ordering(case), port.score_ordering(case))
        assert np.array_equal(tg.permutation_from_scores(case).new_id_of,
                              port.permutation_from_scores(case))


def test_permutation_validation_and_invert(tg, ctx):
    for bad, msg in (([0, 0, 1], "assigned twice"), ([0, 1, 5], "out of range")):
        with pytest.raises(tg.DomainError, match=msg):
            tg.validate_permutation(bad)
        with pytest.raises(tg.DomainError):
            tg.invert(bad)
    p = random_permutation(100_000, 5)
    assert np.array_equal(tg.invert(tg.invert(p)).new_id_of, p)
    assert np.array_equal(tg.invert(p).new_id_of, oracle.port().invert(p))


def test_reorder_features(tg, ctx):
    f = tg.FeatureMatrix(2, 1, 1, np.array([1, 2], np.uint8))  # test_reorder.cpp:122-141
    assert tg.reorder_features(f, [1, 0]).data.tolist() == [2, 1]
    assert tg.reorder_features(f, [0, 1]).data.tolist() == [1, 2]
    with pytest.raises(tg.DomainError):
        tg.reorder_features(f, [0, 1, 2])
    port = oracle.port()
    for rows, dim, eb in ((64, 9, 4), (1000, 3, 1), (5000, 100, 4), (777, 768, 2), (3, 1, 8)):
        data = np.random.default_rng(rows).integers(0, 256, rows * dim * eb, dtype=np.uint8)
        fm = tg.FeatureMatrix(rows, dim, eb, data)
        p = random_permutation(rows, rows + 1)
        got = tg.reorder_features(fm, p)
        want = port.reorder_features(data.reshape(rows, dim * eb), p)
        assert np.array_equal(got.data.reshape(rows, -1), want)
        back = tg.reorder_features(got, tg.invert(p))
        assert np.array_equal(back.data, data)


def test_reorder_graph(tg, ctx):
    port = oracle.port()
    chk = oracle.ref() or port
    g = tg.CsrGraph(*port.from_edge_list(2, np.array([0], np.uint64), np.array([1], np.uint64)))
    out = tg.reorder_graph(g, [1, 0])  # test_reorder.cpp:77-82
    assert list(out.offsets) == [0, 0, 1] and list(out.targets) == [0]
    for i in range(30):  # acceptance.cpp:181-212
        n = 2 + (i * 13) % 199
        off, tgt = random_graph(port, n, 1.0 + i % 5, i)
        p = random_permutation(n, i + 1000)
        got = tg.reorder_graph(tg.CsrGraph(off, tgt), p)
        wo, wt = chk.reorder_graph(off, tgt, p)
        assert np.array_equal(got.offsets, wo) and np.array_equal(got.targets, wt)
    with pytest.raises(tg.DomainError):
        tg.reorder_graph(tg.CsrGraph(*port.from_edge_list(3, np.array([0], np.uint64),
                                                          np.array([1], np.uint64))), [0, 1])
