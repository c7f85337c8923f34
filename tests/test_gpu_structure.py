"""Graph-structure tiering (csrc/structure.cu, SURVEY §8f row 2,
PAPER.md:560-564): the sampler's transposed graph placed by a TierLayout
(replicated / interleaved over D devices / cold in pinned host memory) gives
the SAME build_minibatch lists as the whole graph (sampling.cpp:56-90,
checked against the reference build), and its per-tier neighbour-id reads
equal the C restatement's count (oracle tgo_build_minibatch_tier_reads).
D > 1 runs as D tiered graphs on one GPU wired to each other's slices
(the peer table a multi-GPU node fills with peer pointers)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def checker():
    return oracle.ref() or oracle.port()


def _graph(n, seed, hubs=()):
    port = oracle.port()
    rng = np.random.default_rng(seed)
    src = [rng.integers(0, n, 8 * n)]
    dst = [rng.integers(0, n, 8 * n)]
    for h, length in hubs:
        src.append(rng.choice(n, size=length, replace=False))
        dst.append(np.full(length, h))
    return port.from_edge_list(n, np.concatenate(src).astype(np.uint64),
                               np.concatenate(dst).astype(np.uint64))


def _tiered(tg, producers, go, gt, lay, ctx):
    """D tiered graphs (one per virtual device) sharing one cold tier."""
    D = lay.num_devices
    import ctypes
    gs = [producers.TieredGraph(go, gt, lay, 0, ctx=ctx)]
    nb = producers.TieredGraph.cold_bytes(go, lay)
    cold = np.frombuffer((ctypes.c_uint8 * nb).from_address(gs[0].cold_host), np.uint8)
    for d in range(1, D):  # device 0 wrote the cold rows; the others map them
        gs.append(producers.TieredGraph(go, gt, lay, d, ctx=ctx, cold=cold, fill=False))
    for a in gs:
        for b in gs:
            if a is not b:
                a.set_peer(b.device_index, b.local_base)
    return gs


LAYOUTS = [  # (hot, replicated, D)
    (0.2, 0.0, 1), (0.2, 0.05, 1), (0.3, 0.0, 2), (0.5, 0.1, 3), (0.25, 0.0, 4),
    (1.0, 0.0, 2), (0.0, 0.0, 1), (1.0, 1.0, 1), (0.2, 0.2, 2),
]


@pytest.mark.parametrize("hot,rep,D", LAYOUTS)
def test_tiered_sampler_bit_exact_and_reads(tg, ctx, hot, rep, D):
    from paper_2111_05894_b200 import producers
    chk, port = checker(), oracle.port()
    n = 5000
    off, tgt = _graph(n, int(hot * 100) + D, hubs=[(0, 2500), (3, 400), (4000, 300)])
    go, gt = chk.transpose(off, tgt)
    lay = tg.plan_layout(n, hot, rep, D, 1, 4)
    gs = _tiered(tg, producers, go, gt, lay, ctx)
    tid = port.draw_random_train_ids(n, 700, 3)
    fanouts = [10, 15, 5]
    want = chk.epoch_minibatches(go, gt, tid, fanouts, 64, 7, 0, max_batches=6)
    order = producers.epoch_order(tid, 7, 0)
    for d, g in enumerate(gs):
        s = producers.GpuSampler(g, ctx=ctx)
        for b, w in enumerate(want):
            seeds = order[b * 64:(b + 1) * 64]
            got = s.minibatch(seeds, fanouts, 7, 0, b)
            assert np.array_equal(got, w), f"device {d} batch {b}"
            reads = s.structure_reads(reset=True)
            exp = port.structure_tier_reads(go, gt, seeds, fanouts, lay, d, 7, 0, b)
            assert np.array_equal(reads, exp), (d, b, reads, exp)
        # the same through the back-to-back multi-batch path (sampler lanes)
        got = s.batches(order, fanouts, 64, 7, 0, 0, len(want))
        assert all(np.array_equal(a, w) for a, w in zip(got, want))
        s.close()
    info = gs[0].info()
    lb, mb = lay.local_boundary, lay.multi_boundary
    assert info["replicated_bytes"] == 4 * int(go[lb])
    assert info["host_bytes"] == 4 * int(go[n] - go[mb])
    slices = sum(g.info()["slice_bytes"] for g in gs)
    assert slices == 4 * int(go[mb] - go[lb])
    for g in gs:
        g.close()


def test_tiered_sampler_c1_shape(tg, ctx):
    """C1 shape (R-MAT 200k nodes, score-reordered like the bench), 20 % hot
    sharded over 2 virtual devices: lists equal the whole-graph sampler's and
    the reference's; cold reads are what crosses PCIe."""
    from paper_2111_05894_b200 import producers, synth
    chk = checker()
    off, tgt = synth.rmat_graph(200_000, 3_200_000, seed=1)
    n = len(off) - 1
    tid = oracle.port().draw_random_train_ids(n, n // 10, 3)
    scores = chk.weighted_reverse_pagerank(off, tgt, tid)
    perm = chk.permutation_from_scores(scores)
    ro, rt = chk.reorder_graph(off, tgt, perm)
    go, gt = chk.transpose(ro, rt)
    new_tid = np.sort(perm[tid])
    lay = tg.plan_layout(n, 0.2, 0.0, 2, 1, 4)
    gs = _tiered(tg, producers, go, gt, lay, ctx)
    want = chk.epoch_minibatches(go, gt, new_tid, [10, 15], 1024, 7, 0, max_batches=4)
    order = producers.epoch_order(new_tid, 7, 0)
    whole = producers.GpuSampler(tg.CsrGraph(go, gt), ctx=ctx)
    s = producers.GpuSampler(gs[1], ctx=ctx)
    tot = np.zeros(3, np.uint64)
    for b, w in enumerate(want):
        seeds = order[b * 1024:(b + 1) * 1024]
        got = s.minibatch(seeds, [10, 15], 7, 0, b)
        assert np.array_equal(got, w)
        assert np.array_equal(whole.minibatch(seeds, [10, 15], 7, 0, b), w)
        tot += oracle.port().structure_tier_reads(go, gt, seeds, [10, 15], lay, 1, 7, 0, b)
    assert np.array_equal(s.structure_reads(), tot)
    # hot rows are the high-score (high in-degree) nodes: most reads avoid PCIe
    assert tot[2] < 0.5 * tot.sum()


def test_tiered_graph_errors(tg, ctx):
    from paper_2111_05894_b200 import producers
    off = np.array([0, 1, 3, 3], np.uint64)
    tgt = np.array([2, 0, 1], np.uint64)
    lay = tg.plan_layout(3, 0.5, 0.0, 1, 1, 4)
    with pytest.raises(tg.DomainError, match="out of range"):
        producers.TieredGraph(off, tgt, lay, 1, ctx=ctx)
    with pytest.raises(tg.DomainError, match="layout covers"):
        producers.TieredGraph(off, tgt, tg.plan_layout(4, 0.5, 0.0, 1, 1, 4), 0, ctx=ctx)
    with pytest.raises(tg.FormatError, match="target out of range"):
        producers.TieredGraph(off, np.array([2, 0, 3], np.uint64), lay, 0, ctx=ctx)
    with pytest.raises(tg.FormatError, match="offsets invalid"):
        producers.TieredGraph(np.array([0, 2, 1, 3], np.uint64), tgt, lay, 0, ctx=ctx)
    g = producers.TieredGraph(off, tgt, lay, 0, ctx=ctx)
    with pytest.raises(tg.DomainError, match="out of range"):
        g.set_peer(1, g.local_base)
    s = producers.GpuSampler(tg.CsrGraph(off, tgt), ctx=ctx)
    with pytest.raises(tg.DomainError, match="not tiered"):
        s.structure_reads()
    # a caller-provided cold tier too small
    small = tg.host_alloc(8)
    with pytest.raises(tg.DomainError, match="cold tier needs"):
        producers.TieredGraph(off, tgt, tg.plan_layout(3, 0.0, 0.0, 1, 1, 4), 0, ctx=ctx,
                              cold=small)
