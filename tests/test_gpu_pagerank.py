"""GPU parity: reverse PageRank (K1-K3) is bit-identical to the reference.

Tolerance: none — scores are compared as raw IEEE-754 bytes (the hot set
depends on exact fp64 ties). The checker is the reference build
(oracle/_ref) when present, else the pinned C restatement (oracle/_build).
"""
import numpy as np
import pytest

import oracle
from tests.helpers import RngStream, derive_stream_key, graph_from_pairs, random_graph

pytestmark = pytest.mark.gpu


def checker():
    return oracle.ref() or oracle.port()


def G(tg, off, tgt):
    return tg.CsrGraph(off, tgt)


def test_known_answers(tg, ctx):
    port = oracle.port()
    off, tgt = graph_from_pairs(port, 2, [(0, 1)])  # test_scoring.cpp:27-32
    s = tg.reverse_pagerank(G(tg, off, tgt), tg.PagerankConfig(1, 0.85))
    assert s[0] == pytest.approx(0.5, rel=1e-14) and s[1] == pytest.approx(0.075, rel=1e-14)
    off, tgt = graph_from_pairs(port, 2, [(0, 1), (1, 0)])  # :34-41
    for it in (1, 5, 17):
        s = tg.reverse_pagerank(G(tg, off, tgt), tg.PagerankConfig(it, 0.85))
        assert s[0] == s[1] and s[0] == pytest.approx(0.5, rel=1e-12)
    off, tgt = graph_from_pairs(port, 4, [(2, 0)])  # :74-83 exact dyadic
    s = tg.weighted_reverse_pagerank(G(tg, off, tgt), tg.PagerankConfig(1, 0.5),
                                     tg.TrainIdSet.from_ids([0, 1], 4))
    assert s[2] == 0.375 and s[3] == 0.125
    off, tgt = graph_from_pairs(port, 2, [(0, 1)])  # :85-91
    s = tg.weighted_reverse_pagerank(G(tg, off, tgt), tg.PagerankConfig(1, 0.85),
                                     tg.TrainIdSet.from_ids([0], 2))
    assert s[0] == pytest.approx(0.5, rel=1e-14) and s[1] == pytest.approx(0.075, rel=1e-14)


def test_errors(tg, ctx):
    port = oracle.port()
    g = G(tg, *graph_from_pairs(port, 2, [(0, 1)]))
    with pytest.raises(tg.DomainError):
        tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(np.zeros(0, np.uint64)))
    for it, d in [(0, 0.85), (1, 1.0), (1, 0.0)]:
        with pytest.raises(tg.DomainError):
            tg.reverse_pagerank(g, tg.PagerankConfig(it, d))
    with pytest.raises(tg.DomainError, match="train id 7 out of range"):
        tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(np.array([0, 7], np.uint64)))
    with pytest.raises(tg.FormatError):
        tg.reverse_pagerank(G(tg, np.array([0, 1, 1], np.uint64), np.array([5], np.uint64)))
    # large pageable targets are narrowed by the host cores on the way into
    # the pinned pipeline (copy_h2d_narrow): the first offending edge is still
    # the one reported, whichever chunk or pipeline buffer it falls in
    # (32M-edge chunks: 80M edges = three host-narrowed chunks; 2 x 2^25 + 1000
    # = two host-narrowed chunks and a small tail narrowed on the device)
    n = 1000
    for e, bads in ((80_000_000, ((50_000_001, 79_999_999), (3, 70_000_000), (33_554_431,),
                                  (79_999_999,))),
                    (2 * 2 ** 25 + 1000, ((2 ** 26 + 10,), (100, 2 ** 26 + 999)))):
        off = np.linspace(0, e, n + 1).astype(np.uint64)
        tgt = (np.arange(e, dtype=np.uint64) * np.uint64(7919)) % np.uint64(n)
        for bad in bads:
            t = tgt.copy()
            for i in bad:
                t[i] = n + i % 5
            with pytest.raises(tg.FormatError, match=rf"target out of range at edge {bad[0]}(?!\d)"):
                tg.reverse_pagerank(G(tg, off, t), tg.PagerankConfig(iterations=1))
    # the same graph without bad targets uploads and runs (host-narrowed path)
    s = tg.reverse_pagerank(G(tg, off, tgt), tg.PagerankConfig(iterations=1))
    assert len(s) == n and np.all(np.isfinite(s))
    # empty graph: config still validated, result empty
    e = G(tg, np.zeros(1, np.uint64), np.zeros(0, np.uint64))
    assert tg.reverse_pagerank(e).size == 0
    with pytest.raises(tg.DomainError):
        tg.reverse_pagerank(e, tg.PagerankConfig(0, 0.85))


def test_isolated_and_edgeless(tg, ctx):
    port = oracle.port()
    off, tgt = graph_from_pairs(port, 10, [(0, 1), (2, 1), (3, 4)])
    for s in (tg.reverse_pagerank(G(tg, off, tgt)),
              tg.weighted_reverse_pagerank(G(tg, off, tgt), tg.PagerankConfig(),
                                           tg.TrainIdSet.from_ids([0, 3], 10))):
        assert np.all(np.isfinite(s)) and np.all(s >= 0)
    off = np.zeros(8, np.uint64)
    s = tg.reverse_pagerank(G(tg, off, np.zeros(0, np.uint64)))
    assert s.tobytes() == checker().reverse_pagerank(off, np.zeros(0, np.uint64)).tobytes()


def test_random_graphs_bit_exact(tg, ctx):
    chk, port = checker(), oracle.port()
    for i in range(40):  # acceptance.cpp:112-148 instance mix
        n = 20 + (i * 37) % 481
        off, tgt = random_graph(port, n, 0.5 + i % 8, i)
        g = G(tg, off, tgt)
        tid = port.draw_random_train_ids(n, max(1, n // 10), i)
        for it in (1, 5, 20):
            a = tg.reverse_pagerank(g, tg.PagerankConfig(it, 0.85))
            assert a.tobytes() == chk.reverse_pagerank(off, tgt, it, 0.85).tobytes()
            b = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(it, 0.85), tg.TrainIdSet(tid))
            assert b.tobytes() == chk.weighted_reverse_pagerank(off, tgt, tid, it, 0.85).tobytes()


def test_all_labeled_equals_unweighted(tg, ctx):
    port = oracle.port()
    off, tgt = random_graph(port, 350, 3.0, 7)  # acceptance.cpp:154-162
    g = G(tg, off, tgt)
    a = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(),
                                     tg.TrainIdSet(np.arange(350, dtype=np.uint64)))
    assert a.tobytes() == tg.reverse_pagerank(g).tobytes()


def _hub_graph(n, hubs, seed):
    """Random graph plus hub rows long enough to cross many windows and the
    heavy-group threshold (row lengths 33..40000)."""
    rng = np.random.default_rng(seed)
    src = [rng.integers(0, n, 6 * n)]
    dst = [rng.integers(0, n, 6 * n)]
    for h, length in hubs:
        src.append(np.full(length, h))
        dst.append(rng.choice(n, size=length, replace=False))
    src = np.concatenate(src).astype(np.uint64)
    dst = np.concatenate(dst).astype(np.uint64)
    return oracle.port().from_edge_list(n, src, dst)


def test_long_rows_and_heavy_groups(tg, ctx):
    chk = checker()
    n = 60000
    hubs = [(0, 40000), (1, 257), (31, 2049), (32, 5000), (95, 33), (1000, 20000), (59999, 3000),
            (2, 45000), (3, 58000)]
    off, tgt = _hub_graph(n, hubs, 3)
    g = G(tg, off, tgt)
    tid = oracle.port().draw_random_train_ids(n, 600, 5)
    for it in (1, 5):
        a = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(it, 0.85), tg.TrainIdSet(tid))
        assert a.tobytes() == chk.weighted_reverse_pagerank(off, tgt, tid, it, 0.85).tobytes()


def test_in_degrees_and_degree_score(tg, ctx):
    port = oracle.port()
    off, tgt = _hub_graph(20000, [(0, 15000), (7, 100)], 9)
    g = G(tg, off, tgt)
    assert np.array_equal(tg.in_degrees(g), port.in_degrees(off, tgt))
    assert np.array_equal(tg.degree_score(g), port.degree_score(off))


def test_row_partitioned_steps_equal_full_run(tg, ctx):
    """The multi-GPU decomposition (row blocks + all-gather of `norm`) run as
    several row ranges on one device reproduces the single run bit for bit."""
    import torch
    from paper_2111_05894_b200._lib import LIB
    port = oracle.port()
    n = 5000
    off, tgt = _hub_graph(n, [(3, 3000), (64, 900)], 11)
    g = G(tg, off, tgt)
    tid = port.draw_random_train_ids(n, 400, 1)
    want = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(5, 0.85), tg.TrainIdSet(tid))
    dev = torch.device("cuda", ctx.device)
    tid_d = torch.as_tensor(tid.astype(np.int64), device=dev)
    deg = torch.empty(n, dtype=torch.int32, device=dev)
    na = torch.empty(n, dtype=torch.float64, device=dev)
    nb = torch.empty_like(na)
    score = torch.empty_like(na)
    gh = g.device(ctx)
    assert LIB.tg_pagerank_prepare_async(ctx.h, gh, tid_d.data_ptr(), len(tid),
                                         deg.data_ptr(), na.data_ptr()) == 0
    bounds = [0, 32 * 20, 32 * 61, 32 * 100, n]  # 4 "ranks", 32-row aligned
    for it in range(5):
        last = int(it == 4)
        for r0, r1 in zip(bounds[:-1], bounds[1:]):
            assert LIB.tg_pagerank_step_async(ctx.h, gh, deg.data_ptr(), 0.85, na.data_ptr(),
                                              nb.data_ptr(), score.data_ptr(), r0, r1, last) == 0
        na, nb = nb, na
    ctx.sync()
    assert score.cpu().numpy().tobytes() == want.tobytes()


def test_rmat_c1_scale_bit_exact_and_hot_set(tg, ctx):
    """C1 shape (R-MAT 1M nodes / 16M draws, 10 % train): bit-exact scores and
    an identical hot set / permutation (the tie-break by id included)."""
    from paper_2111_05894_b200 import synth
    off, tgt = synth.rmat_graph(1_000_000, 16_000_000, seed=1)
    port = oracle.port()
    tid = port.draw_random_train_ids(1_000_000, 100_000, 3)
    g = G(tg, off, tgt)
    got = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(tid))
    want = port.weighted_reverse_pagerank(off, tgt, tid)
    assert got.tobytes() == want.tobytes()
    perm = tg.permutation_from_scores(got)
    assert np.array_equal(perm.new_id_of, port.permutation_from_scores(want))


def test_hub_rows_with_tie_prone_addends(tg, ctx):
    """Hub rows (> 2048 edges, the parallel exact-chain path) whose addends are
    all equal or few-valued, so the running sum hits round-half-even ties and
    binade crossings at many points: still bit-identical to the serial sum."""
    chk = checker()
    port = oracle.port()
    n = 3 * 2 ** 15
    src = [np.zeros(60000, np.uint64), np.ones(n - 60001, np.uint64),
           np.full(5000, 2, np.uint64)]
    dst = [np.arange(1, 60001, dtype=np.uint64), np.arange(60001, n, dtype=np.uint64),
           np.random.default_rng(4).choice(n, 5000, replace=False).astype(np.uint64)]
    off, tgt = port.from_edge_list(n, np.concatenate(src), np.concatenate(dst))
    g = G(tg, off, tgt)
    for tid in (np.arange(0, n, 3, dtype=np.uint64), np.arange(n, dtype=np.uint64)):
        for it in (1, 2, 5):
            a = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(it, 0.85), tg.TrainIdSet(tid))
            assert a.tobytes() == chk.weighted_reverse_pagerank(off, tgt, tid, it, 0.85).tobytes()
    a = tg.reverse_pagerank(g, tg.PagerankConfig(3, 0.5))
    assert a.tobytes() == chk.reverse_pagerank(off, tgt, 3, 0.5).tobytes()


def test_partitioned_driver_single_rank_on_device(tg, ctx):
    """distributed.weighted_reverse_pagerank_multi (DeviceStepper) without a
    process group equals the single call bit for bit."""
    from paper_2111_05894_b200 import distributed as D
    port = oracle.port()
    n = 20000
    off, tgt = _hub_graph(n, [(0, 9000), (5, 3000)], 21)
    g = G(tg, off, tgt)
    tid = port.draw_random_train_ids(n, 2000, 4)
    want = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(tid))
    got = D.weighted_reverse_pagerank_multi(g, tg.PagerankConfig(), tg.TrainIdSet(tid), ctx=ctx)
    assert got.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("ranks", [2, 3, 4])
def test_fused_peer_exchange_virtual_ranks(tg, ctx, ranks):
    """The fused exchange (rows stored straight into every rank's `norm`, a
    device barrier instead of the all-gather) with `ranks` contexts on one
    GPU: every rank ends with the single-GPU scores, bit for bit."""
    from paper_2111_05894_b200 import distributed as D
    port = oracle.port()
    n = 12000
    off, tgt = _hub_graph(n, [(0, 9000), (4000, 5000), (11999, 3000)], 31)
    g = G(tg, off, tgt)
    tid = port.draw_random_train_ids(n, 1200, 2)
    want = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(tid))
    ctxs = [tg.Context(ctx.device) for _ in range(ranks)]
    outs = D.weighted_reverse_pagerank_peers(g, tg.PagerankConfig(), tg.TrainIdSet(tid), ctxs)
    for o in outs:
        assert o.cpu().numpy().tobytes() == want.tobytes()
    un = D.weighted_reverse_pagerank_peers(g, tg.PagerankConfig(3, 0.85), None, ctxs)
    want_un = tg.reverse_pagerank(g, tg.PagerankConfig(3, 0.85))
    assert all(o.cpu().numpy().tobytes() == want_un.tobytes() for o in un)


@pytest.mark.parametrize("k1", ["", "atomic", "bs17"])
@pytest.mark.parametrize("n,draws", [(200_000, 5_000_000), (1_500_000, 6_000_000),
                                     (6_000_000, 8_000_000)])
def test_in_degrees_large_graphs(tg, ctx, monkeypatch, n, draws, k1):
    """K1 on graphs with >= 4M edges (R-MAT hubs, privatised low ids, one id
    holding 1.5M edges) equals csr_graph.cpp:89-93 exactly, in both forms:
    binned (partition + shared-memory histograms, the default at these sizes;
    the 1.5M-edge bucket is split over histogram pieces; 184 buckets at 6M
    nodes; TIERGRAPH_K1_BS=17: 2^17-id buckets, each piece counted by four
    CTAs over their own ranges, the C3 shape) and one-pass atomic
    (TIERGRAPH_K1=atomic)."""
    from paper_2111_05894_b200 import synth
    monkeypatch.delenv("TIERGRAPH_K1", raising=False)
    monkeypatch.delenv("TIERGRAPH_K1_BS", raising=False)
    if k1 == "bs17":  # 2^17-id buckets, four histogram CTAs per piece (the C3 shape)
        monkeypatch.setenv("TIERGRAPH_K1_BS", "17")
    elif k1:
        monkeypatch.setenv("TIERGRAPH_K1", k1)
    off, tgt = synth.rmat_graph(n, draws, seed=11)
    assert len(tgt) >= 1 << 22
    want = np.bincount(tgt.astype(np.int64), minlength=n).astype(np.uint64)
    g = tg.CsrGraph(off, tgt)
    assert np.array_equal(tg.in_degrees(g, ctx=ctx), want)
    # a hub id holding more than one count item (> 2^20 edges) and an empty tail
    tgt2 = np.sort(np.concatenate([np.zeros(1_500_000, np.uint64),
                                   np.random.default_rng(1).integers(0, n // 2, 3_000_000)
                                   .astype(np.uint64)]))
    off2 = np.zeros(n + 1, np.uint64)
    off2[1:] = len(tgt2)  # one row holds every edge (unsorted rows are fine for K1)
    g2 = tg.CsrGraph(off2, tgt2)
    want2 = np.bincount(tgt2.astype(np.int64), minlength=n).astype(np.uint64)
    assert np.array_equal(tg.in_degrees(g2, ctx=ctx), want2)


@pytest.mark.parametrize("mode,cstream,label", [("1", "1", ""), ("1", "0", ""), ("0", "1", ""),
                                                ("1", "0", "indeg"), ("1", "0", "rows"),
                                                ("1", "1", "indeg")])
def test_relabelled_twin_bit_exact(tg, ctx, monkeypatch, mode, cstream, label):
    """K3 on the relabelled twin (TIERGRAPH_PR_RELABEL=1, the default at C3/C4
    sizes; labels by TIERGRAPH_PR_LABEL: hybrid (default), indeg, rows) and
    without it (=0): raw-byte equal to the reference on random, hub-row,
    tie-prone and R-MAT graphs, weighted and plain, and the timed entry point
    returns the same bytes."""
    import ctypes as C
    from paper_2111_05894_b200._lib import LIB
    from paper_2111_05894_b200 import synth
    monkeypatch.setenv("TIERGRAPH_PR_RELABEL", mode)
    monkeypatch.setenv("TIERGRAPH_PR_CSTREAM", cstream)  # streamed class C (twin only)
    monkeypatch.setenv("TIERGRAPH_PR_LABEL", label)
    chk, port = checker(), oracle.port()
    cases = [random_graph(port, 300 + 97 * i, 1.5 + i, 40 + i) for i in range(4)]
    cases.append(_hub_graph(60000, [(0, 40000), (31, 2049), (1000, 20000), (59999, 3000)], 3))
    n = 3 * 2 ** 15
    src = [np.zeros(60000, np.uint64), np.ones(n - 60001, np.uint64)]
    dst = [np.arange(1, 60001, dtype=np.uint64), np.arange(60001, n, dtype=np.uint64)]
    cases.append(port.from_edge_list(n, np.concatenate(src), np.concatenate(dst)))
    cases.append(synth.rmat_graph(300_000, 4_000_000, seed=5))
    for off, tgt in cases:
        nn = len(off) - 1
        g = G(tg, off, tgt)
        info = C.c_int()
        assert LIB.tg_pagerank_relabel_info(ctx.h, g.device(ctx), C.byref(info), None) == 0
        assert info.value == int(mode)
        tid = port.draw_random_train_ids(nn, max(1, nn // 10), 9)
        for it in (1, 5):
            a = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(it, 0.85), tg.TrainIdSet(tid))
            assert a.tobytes() == chk.weighted_reverse_pagerank(off, tgt, tid, it, 0.85).tobytes()
        b = tg.reverse_pagerank(g, tg.PagerankConfig(3, 0.85))
        assert b.tobytes() == chk.reverse_pagerank(off, tgt, 3, 0.85).tobytes()
        out = np.empty(nn, np.float64)
        ph = (C.c_double * 6)()
        t = np.ascontiguousarray(tid, np.uint64)
        assert LIB.tg_weighted_reverse_pagerank_timed(ctx.h, g.device(ctx), 5, 0.85, t.ctypes.data,
                                                      len(t), out.ctypes.data, ph) == 0
        assert out.tobytes() == chk.weighted_reverse_pagerank(off, tgt, tid, 5, 0.85).tobytes()
        assert all(x > 0 for x in ph)
    # out-of-range train ids are still a DomainError on the twin
    g = G(tg, *cases[0])
    with pytest.raises(tg.DomainError, match="out of range"):
        tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(np.array([0, 10 ** 6], np.uint64)))
