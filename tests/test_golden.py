"""Golden vectors from the UNMODIFIED reference build (tests/golden/golden_small.npz,
made by tests/golden/make_golden.py from oracle/_ref): every hot-path output
of a small BA graph and a hub-row graph, as the reference computed them.

CPU: the plain-C restatement (oracle/_build) reproduces every golden array, so
the oracle is pinned to the reference even where /root/reference is absent.
GPU: this library reproduces them through its public API — PageRank scores as
raw IEEE bytes, the permutation, the reordered graph and its transpose, the
sampler's minibatch lists, gathered rows (sha256) and TrafficReports for
1-3 devices, the hot-fraction sweep, in-degrees.
"""
import hashlib
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_small.npz")


@pytest.fixture(scope="module")
def g():
    return dict(np.load(GOLDEN))


def _lists(g):
    out, o = [], 0
    for n in g["list_lens"].astype(np.int64):
        out.append(g["lists"][o:o + n])
        o += n
    return out


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)


LAYOUTS = [(0.2, 0.0, 1), (0.3, 0.05, 2), (0.5, 0.1, 3)]


# ------------------------------------------------------------------- CPU
def test_port_reproduces_golden(g):
    """The restatement (tg_oracle.c) against the reference's own outputs."""
    port = oracle.port()
    N, M, SEED, TRAIN, DIM, BATCH, NB = (int(x) for x in g["params"])
    off, tgt = g["off"], g["tgt"]
    assert np.array_equal(port.draw_random_train_ids(N, TRAIN, 3), g["tid"])
    assert np.array_equal(port.in_degrees(off, tgt), g["indeg"])
    s = port.weighted_reverse_pagerank(off, tgt, g["tid"])
    assert s.tobytes() == g["scores"].tobytes()
    perm = port.permutation_from_scores(s)
    assert np.array_equal(perm, g["perm"])
    ro, rt = port.reorder_graph(off, tgt, perm)
    go, gt = port.transpose(ro, rt)
    assert np.array_equal(go, g["goff"]) and np.array_equal(gt, g["gtgt"])
    lists = port.epoch_minibatches(go, gt, np.sort(perm[g["tid"]]), list(g["fanouts"]), BATCH, 7, 0,
                                   max_batches=NB)
    assert all(np.array_equal(a, b) for a, b in zip(lists, _lists(g)))
    feat = port.make_test_features(N, DIM)
    re = port.reorder_features(feat, perm)
    for x, h in zip(lists, g["rows_sha256"]):
        assert np.array_equal(_sha(re[x.astype(np.int64)]), h)
    k = 0
    for lay, (hot, rep, d) in zip(g["layouts"], LAYOUTS):
        assert tuple(int(v) for v in lay) == port.plan_layout(N, hot, rep, d, DIM, 4)
        for x in lists:
            for dev in range(d):
                assert np.array_equal(port.gather(lay, x, dev), g["reports"][k])
                k += 1
    sl, sr, sf = port.hot_fraction_sweep(g["counts_old"], g["order"], g["fractions"], 0.05, 2, DIM, 4)
    assert np.array_equal(sl, g["sweep_layouts"]) and np.array_equal(sr, g["sweep_reports"])
    assert np.array_equal(sf, g["sweep_rep"])
    s2 = port.weighted_reverse_pagerank(g["off2"], g["tgt2"], g["tid2"])
    assert s2.tobytes() == g["scores2"].tobytes()
    assert port.reverse_pagerank(g["off2"], g["tgt2"], 7, 0.5).tobytes() == g["scores2_plain"].tobytes()
    assert np.array_equal(port.permutation_from_scores(s2), g["perm2"])


# ------------------------------------------------------------------- GPU
def _virtual_devices(tg, ctx, feat, perm, lay):
    D = lay.num_devices
    st = [tg.TieredFeatureStore(feat, perm, lay, d, ctx=ctx, place=False) for d in range(D)]
    for d in range(1, D):
        st[d].share_cold(st[0])
    for s in st:
        s.place(feat, perm)
    for s in st:
        for d in range(D):
            if d != s.device_index:
                s.set_peer(d, st[d].local_base)
    return st


@pytest.mark.gpu
def test_gpu_reproduces_golden(tg, ctx, g):
    from paper_2111_05894_b200 import producers, synth
    N, M, SEED, TRAIN, DIM, BATCH, NB = (int(x) for x in g["params"])
    graph = tg.CsrGraph(g["off"], g["tgt"])
    assert np.array_equal(np.asarray(tg.in_degrees(graph, ctx=ctx), np.uint64), g["indeg"])
    s = tg.weighted_reverse_pagerank(graph, tg.PagerankConfig(), tg.TrainIdSet(g["tid"]), ctx=ctx)
    assert s.tobytes() == g["scores"].tobytes()
    perm = tg.permutation_from_scores(s, ctx=ctx)
    assert np.array_equal(perm.new_id_of, g["perm"])
    rg = tg.reorder_graph(graph, perm, ctx=ctx)
    gt = tg.transpose(rg, ctx=ctx)
    assert np.array_equal(gt.offsets, g["goff"]) and np.array_equal(gt.targets, g["gtgt"])
    sampler = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(np.sort(perm.new_id_of[g["tid"]]), 7, 0)
    lists = sampler.batches(order, list(g["fanouts"]), BATCH, 7, 0, 0, NB)
    assert all(np.array_equal(a, b) for a, b in zip(lists, _lists(g)))
    feat = synth.test_features(N, DIM)
    k = 0
    for lay_g, (hot, rep, d) in zip(g["layouts"], LAYOUTS):
        lay = tg.plan_layout(N, hot, rep, d, DIM, 4)
        assert lay.as_tuple() == tuple(int(v) for v in lay_g)
        stores = _virtual_devices(tg, ctx, feat, perm, lay)
        for x, h in zip(lists, g["rows_sha256"]):
            for dev, st in enumerate(stores):
                r = tg.TrafficReport()
                rows = st.gather_rows(x, report=r)
                assert np.array_equal(_sha(rows), h)
                assert np.array_equal(r.as_array(), g["reports"][k])
                k += 1
    rows = tg.hot_fraction_sweep(tg.make_access_counter(g["counts_old"]), g["order"],
                                 list(g["fractions"]), 0.05, 2, DIM, 4, ctx=ctx)
    for r, lay, rep, rf in zip(rows, g["sweep_layouts"], g["sweep_reports"], g["sweep_rep"]):
        assert r.layout.as_tuple() == tuple(int(v) for v in lay)
        assert np.array_equal(r.report.as_array(), rep) and r.replicated_fraction == rf
    g2 = tg.CsrGraph(g["off2"], g["tgt2"])
    s2 = tg.weighted_reverse_pagerank(g2, tg.PagerankConfig(), tg.TrainIdSet(g["tid2"]), ctx=ctx)
    assert s2.tobytes() == g["scores2"].tobytes()
    assert tg.reverse_pagerank(g2, tg.PagerankConfig(7, 0.5), ctx=ctx).tobytes() == \
        g["scores2_plain"].tobytes()
    assert np.array_equal(tg.permutation_from_scores(s2, ctx=ctx).new_id_of, g["perm2"])
