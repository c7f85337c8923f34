"""Pin the CPU oracle (tg_oracle.c) before trusting it.

Every known answer below is one the reference's own tests assert (cited), run
against BOTH the restatement and the reference build; then the restatement is
checked bit-for-bit against the reference build on seeded random inputs.
CPU only.
"""
import numpy as np
import pytest

import oracle
from tests.helpers import (RngStream, dense_reverse_pagerank, derive_stream_key, graph_from_pairs,
                           mix64, random_counter, random_graph, random_layout, random_permutation)


def oracles():
    out = [oracle.port()]
    r = oracle.ref()
    if r is not None:
        out.append(r)
    return out


@pytest.fixture(params=["port", "reference"])
def orc(request):
    if request.param == "port":
        return oracle.port()
    r = oracle.ref()
    if r is None:
        pytest.skip("reference build not present")
    return r


LISTING = (16, 4, 10, 2, 8, 4)  # tests/test_tiering.cpp:15-24


# ---------------------------------------------------------------- rng
def test_rng_matches_python_restatement(orc):
    for x in [0, 1, 0xDEADBEEF, (1 << 64) - 1]:
        assert orc.mix64(x) == mix64(x)
    assert orc.derive_stream_key(7, [1, 2, 3]) == derive_stream_key(7, [1, 2, 3])


# ---------------------------------------------------------------- pagerank
def test_pagerank_single_edge_one_iteration(orc):  # test_scoring.cpp:27-32
    off, tgt = graph_from_pairs(orc, 2, [(0, 1)])
    s = orc.reverse_pagerank(off, tgt, 1, 0.85)
    assert s[0] == pytest.approx(0.5, rel=1e-14)
    assert s[1] == pytest.approx(0.075, rel=1e-14)


def test_pagerank_two_cycle(orc):  # test_scoring.cpp:34-41
    off, tgt = graph_from_pairs(orc, 2, [(0, 1), (1, 0)])
    for it in (1, 5, 17):
        s = orc.reverse_pagerank(off, tgt, it, 0.85)
        assert s[0] == s[1]
        assert s[0] == pytest.approx(0.5, rel=1e-12)


def test_pagerank_dense_oracle(orc):  # test_scoring.cpp:43-53 ; acceptance.cpp:112-148
    for seed in range(3):
        off, tgt = random_graph(orc, 60 + 40 * seed, 2.5, seed)
        for it in (1, 5, 20):
            got = orc.reverse_pagerank(off, tgt, it, 0.85)
            want = dense_reverse_pagerank(off, tgt, it, 0.85)
            assert np.max(np.abs(got - want)) <= 1e-12


def test_weighted_dyadic(orc):  # test_scoring.cpp:74-83 ; acceptance.cpp:168-174
    off, tgt = graph_from_pairs(orc, 4, [(2, 0)])
    s = orc.weighted_reverse_pagerank(off, tgt, [0, 1], 1, 0.5)
    assert s[2] == 0.375 and s[3] == 0.125


def test_weighted_single_edge(orc):  # test_scoring.cpp:85-91
    off, tgt = graph_from_pairs(orc, 2, [(0, 1)])
    s = orc.weighted_reverse_pagerank(off, tgt, [0], 1, 0.85)
    assert s[0] == pytest.approx(0.5, rel=1e-14) and s[1] == pytest.approx(0.075, rel=1e-14)


def test_weighted_all_labeled_bit_identical(orc):  # test_scoring.cpp:93-100
    off, tgt = random_graph(orc, 150, 3.0, 2)
    a = orc.weighted_reverse_pagerank(off, tgt, np.arange(150, dtype=np.uint64))
    b = orc.reverse_pagerank(off, tgt)
    assert a.tobytes() == b.tobytes()


def test_weighted_dense_oracle(orc):  # test_scoring.cpp:102-110
    off, tgt = random_graph(orc, 120, 3.0, 4)
    lab = [3, 17, 44, 90]
    got = orc.weighted_reverse_pagerank(off, tgt, lab, 5, 0.85)
    want = dense_reverse_pagerank(off, tgt, 5, 0.85, lab)
    assert np.max(np.abs(got - want)) <= 1e-12


def test_pagerank_errors(orc):  # test_scoring.cpp:112-115, 151-156
    off, tgt = graph_from_pairs(orc, 2, [(0, 1)])
    with pytest.raises(oracle.DomainError):
        orc.weighted_reverse_pagerank(off, tgt, [], 5, 0.85)
    for it, d in [(0, 0.85), (1, 1.0), (1, 0.0)]:
        with pytest.raises(oracle.DomainError):
            orc.reverse_pagerank(off, tgt, it, d)


def test_isolated_and_sinks_finite(orc):  # test_scoring.cpp:117-129
    off, tgt = graph_from_pairs(orc, 10, [(0, 1), (2, 1), (3, 4)])
    for s in (orc.reverse_pagerank(off, tgt), orc.weighted_reverse_pagerank(off, tgt, [0, 3])):
        assert np.all(np.isfinite(s)) and np.all(s >= 0)


# ---------------------------------------------------------------- ordering
def test_score_ordering_examples(orc):  # test_scoring.cpp:145-149
    assert list(orc.score_ordering([0.1, 0.4, 0.2, 0.3])) == [1, 3, 2, 0]
    assert list(orc.score_ordering([7.0, 7.0, 7.0])) == [0, 1, 2]
    assert list(orc.score_ordering([5.0, 5.0, 1.0])) == [0, 1, 2]


def test_score_ordering_rejects(orc):  # scoring.cpp:105-107
    for bad in ([0.1, float("nan")], [float("inf")], [-1e-300]):
        with pytest.raises(oracle.DomainError):
            orc.score_ordering(bad)
    # -0.0 == +0.0: ties broken by id (scoring.cpp:111)
    assert list(orc.score_ordering([0.0, -0.0, 0.0])) == [0, 1, 2]


def test_permutation_examples(orc):  # test_reorder.cpp:42-60 ; acceptance.cpp:182-184
    assert list(orc.permutation_from_scores([0.1, 0.4, 0.2, 0.3])) == [3, 0, 2, 1]
    assert list(orc.permutation_from_scores([9.0, 8.0, 7.0])) == [0, 1, 2]
    assert list(orc.permutation_from_scores([1.0, 1.0, 1.0])) == [0, 1, 2]
    s = [0.3, 0.9, 0.9, 0.1, 0.5]
    order, perm = orc.score_ordering(s), orc.permutation_from_scores(s)
    assert all(perm[order[r]] == r for r in range(5))


def test_invert_examples(orc):  # test_reorder.cpp:62-67
    assert list(orc.invert([0, 1, 2])) == [0, 1, 2]
    assert list(orc.invert([3, 0, 2, 1])) == [1, 3, 2, 0]
    p = random_permutation(40, 5)
    assert np.array_equal(orc.invert(orc.invert(p)), p)
    with pytest.raises(oracle.DomainError):
        orc.invert([0, 0, 1])


# ---------------------------------------------------------------- reorder
def test_reorder_graph_examples(orc):  # test_reorder.cpp:69-82, 115-120
    off, tgt = graph_from_pairs(orc, 2, [(0, 1)])
    o, t = orc.reorder_graph(off, tgt, [1, 0])
    assert list(o) == [0, 0, 1] and list(t) == [0]
    off, tgt = random_graph(orc, 50, 3.0, 1)
    o, t = orc.reorder_graph(off, tgt, np.arange(50, dtype=np.uint64))
    assert np.array_equal(o, off) and np.array_equal(t, tgt)
    off, tgt = graph_from_pairs(orc, 3, [(0, 1)])
    for bad in ([0, 0, 1], [0, 1, 5], [0, 1]):
        with pytest.raises(oracle.DomainError):
            orc.reorder_graph(off, tgt, bad)


def test_reorder_features_examples(orc):  # test_reorder.cpp:122-141
    f = np.array([[1], [2]], np.uint8)
    assert orc.reorder_features(f, [1, 0]).ravel().tolist() == [2, 1]
    assert orc.reorder_features(f, [0, 1]).ravel().tolist() == [1, 2]
    big = orc.make_test_features(64, 9)
    p = random_permutation(64, 3)
    assert np.array_equal(orc.reorder_features(orc.reorder_features(big, p), orc.invert(p)), big)
    with pytest.raises(oracle.DomainError):
        orc.reorder_features(f, [0, 1, 2])


def test_make_test_features_closed_form(orc):  # feature_matrix.cpp:16-28
    f = orc.make_test_features(5, 3)
    for r in range(5):
        for c in range(3):
            assert f[r, c] == np.float32(np.float32(mix64(r) >> 40) + np.float32(c))


# ---------------------------------------------------------------- tiering
def test_resolve_listing(orc):  # test_tiering.cpp:39-50 ; acceptance.cpp:445-450
    assert orc.resolve(LISTING, 2, 0) == (0, 0, 2)
    assert orc.resolve(LISTING, 5, 0) == (1, 1, 0)
    assert orc.resolve(LISTING, 11, 0) == (2, 0, 1)
    with pytest.raises(oracle.DomainError):
        orc.resolve(LISTING, 16, 0)
    with pytest.raises(oracle.DomainError):
        orc.resolve(LISTING, 0, 2)


def test_plan_layout_examples(orc):  # test_tiering.cpp:95-122
    l = orc.plan_layout(100, 0.10, 0.05, 4, 8, 4)
    assert l[1] == 5 and l[2] == 10
    assert orc.plan_layout(100, 0.0, 0.0, 2, 8, 4)[2] == 0
    hot = orc.plan_layout(100, 1.0, 0.0, 1, 8, 4)
    assert hot[1] == 0 and hot[2] == 100
    with pytest.raises(oracle.DomainError):
        orc.plan_layout(100, 0.5, 0.1, 4, 8, 4, 639)
    assert orc.plan_layout(100, 0.5, 0.1, 4, 8, 4, 640)[2] == 50
    with pytest.raises(oracle.DomainError):
        orc.plan_layout(100, 0.2, 0.5, 4, 8, 4)


def test_gather_accounting_examples(orc):  # test_tiering.cpp:124-153
    rb = 32
    r = orc.gather(LISTING, [0, 1, 3], 0)
    assert r[5] == 0 and r[0] == 3 and r[3] == 3 * rb
    cold = (16, 0, 0, 2, 8, 4)
    r = orc.gather(cold, [0, 5, 11, 15], 1)
    assert r[2] == 4 and r[5] == 4 * rb and r[0] + r[1] == 0
    r = orc.gather(LISTING, [2, 5, 11], 0)
    assert (r[0], r[1], r[2]) == (1, 1, 1)
    assert orc.gather(LISTING, [5], 1)[0] == 1


def test_simulate_trace_examples(orc):  # test_tiering.cpp:155-174
    lay = (3, 0, 1, 1, 2, 4)
    r = orc.simulate_trace([5, 3, 2], lay)
    assert r[5] == 5 * 8 and r[2] == 5 and r[0] == 5
    r = orc.simulate_trace([5, 3, 2], (3, 0, 3, 1, 2, 4))
    assert r[5] == 0
    with pytest.raises(oracle.DomainError):
        orc.simulate_trace([0, 0], (2, 0, 1, 1, 1, 4))
    with pytest.raises(oracle.DomainError):
        orc.simulate_trace([1, 1, 1], (2, 0, 1, 1, 1, 4))


def test_sweep_endpoints(orc):  # test_tiering.cpp:225-243
    counts = np.array([9, 1, 4, 0, 2, 7, 3, 3, 1, 5], np.uint64)
    ordering = orc.score_ordering(counts.astype(np.float64))
    lays, reps, _ = orc.hot_fraction_sweep(counts, ordering, [0.0, 0.25, 0.5, 0.75, 1.0], 0.0, 2, 4, 4)
    assert reps[0][0] + reps[0][1] == 0 and reps[-1][2] == 0
    assert all(reps[i][5] <= reps[i - 1][5] for i in range(1, 5))
    with pytest.raises(oracle.DomainError):
        orc.hot_fraction_sweep(counts, ordering, [0.5, 0.1], 0.0, 2, 4, 4)


# ---------------------------------------------------------------- sampling
def test_build_minibatch_examples(orc):  # test_sampling.cpp build_minibatch cases
    off, tgt = graph_from_pairs(orc, 3, [(0, 1)])
    go, gt = orc.transpose(off, tgt)
    assert list(orc.build_minibatch(go, gt, [2], [10, 10])) == [2]
    off, tgt = graph_from_pairs(orc, 3, [(0, 1), (1, 2)])
    go, gt = orc.transpose(off, tgt)
    assert list(orc.build_minibatch(go, gt, [2], [1, 1])) == [0, 1, 2]
    with pytest.raises(oracle.DomainError):
        orc.build_minibatch(go, gt, [], [1])


# ------------------------------------------------- restatement == reference
def _need_ref():
    r = oracle.ref()
    if r is None:
        pytest.skip("reference build not present")
    return r


def test_port_equals_reference_random_graphs():
    ref, port = _need_ref(), oracle.port()
    for seed in range(12):
        n = 20 + 37 * seed
        off, tgt = random_graph(port, n, 0.5 + seed % 8, seed)
        o2, t2 = ref.from_edge_list(n, *_edges(off, tgt))
        assert np.array_equal(off, o2) and np.array_equal(t2, tgt)
        assert np.array_equal(port.in_degrees(off, tgt), ref.in_degrees(off, tgt))
        tid = port.draw_random_train_ids(n, max(1, n // 10), seed)
        assert np.array_equal(tid, ref.draw_random_train_ids(n, max(1, n // 10), seed))
        for it in (1, 5, 20):
            a = port.weighted_reverse_pagerank(off, tgt, tid, it, 0.85)
            b = ref.weighted_reverse_pagerank(off, tgt, tid, it, 0.85)
            assert a.tobytes() == b.tobytes()
        s = port.weighted_reverse_pagerank(off, tgt, tid)
        assert np.array_equal(port.score_ordering(s), ref.score_ordering(s))
        p = port.permutation_from_scores(s)
        assert np.array_equal(p, ref.permutation_from_scores(s))
        ro, rt = port.reorder_graph(off, tgt, p)
        ro2, rt2 = ref.reorder_graph(off, tgt, p)
        assert np.array_equal(ro, ro2) and np.array_equal(rt, rt2)
        go, gt = port.transpose(ro, rt)
        go2, gt2 = ref.transpose(ro, rt)
        assert np.array_equal(go, go2) and np.array_equal(gt, gt2)
        seeds = port.permutation_from_scores(s)[tid][: 16]
        for fan in ([3], [10, 15], [15, 10, 5], [70, 2]):
            a = port.build_minibatch(go, gt, seeds, fan, 7, 1, seed)
            b = ref.build_minibatch(go, gt, seeds, fan, 7, 1, seed)
            assert np.array_equal(a, b)


def _edges(off, tgt):
    n = len(off) - 1
    src = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off).astype(np.int64))
    return src, tgt


def test_port_equals_reference_tiering_random():
    ref, port = _need_ref(), oracle.port()
    for i in range(60):  # acceptance.cpp:384-411 style instances
        rng = RngStream(derive_stream_key(i, [0xACC7]))
        n = 1 + rng.next_below(300)
        lay = random_layout(rng, n)
        counts = random_counter(n, i, tag=0x636E, bound=25)
        assert np.array_equal(port.simulate_trace(counts, lay), ref.simulate_trace(counts, lay))
        ids = np.array([rng.next_below(n) for _ in range(50)], np.uint64)
        for dev in range(lay[3]):
            assert np.array_equal(port.gather(lay, ids, dev), ref.gather(lay, ids, dev))
        for row in range(0, n, 7):
            assert port.resolve(lay, row, 0) == ref.resolve(lay, row, 0)
        ordering = port.score_ordering(counts.astype(np.float64))
        fr = [0.0, 0.05, 0.1, 0.25, 0.5, 1.0]
        a = port.hot_fraction_sweep(counts, ordering, fr, 0.1, lay[3], 8, 4)
        b = ref.hot_fraction_sweep(counts, ordering, fr, 0.1, lay[3], 8, 4)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_port_plan_layout_rounding_matches_reference():
    ref, port = _need_ref(), oracle.port()
    for n in (1, 3, 7, 10, 999, 1_000_000, 2_449_029, 111_059_956):
        for f in (0.0, 0.05, 0.1, 0.125, 0.2, 0.25, 0.5, 0.55, 1.0):
            for d in (1, 2, 3, 8):
                assert port.plan_layout(n, f, f / 2, d, 128, 4) == ref.plan_layout(n, f, f / 2, d, 128, 4)
