"""GPU parity at config scale (C2: ogbn-products-shaped R-MAT, 2.45M nodes,
47.3M edges after dedup, 100-d f32) against the unmodified reference build
(oracle/_ref) on the same inputs:

* weighted reverse PageRank: raw fp64 bytes (no tolerance);
* the permutation (score order, ties by id);
* reorder_graph + transpose: identical CSR;
* the GPU sampler: the epoch's first minibatches identical to the
  reference's build_minibatch lists;
* K8 tiered gather of one minibatch: rows byte-exact against the reference's
  FeatureMatrix::row of reorder_features' copy, TrafficReport equal to the
  reference gather().
"""
import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu]

N, DRAWS, DIM = 2_450_000, 61_900_000, 100


@pytest.fixture(scope="module")
def c2(ref, tg, ctx):
    from paper_2111_05894_b200 import synth
    off, tgt = synth.rmat_graph(N, DRAWS, seed=1, device="cuda")
    tid = ref.draw_random_train_ids(N, N // 10, 3)
    return off, tgt, tid


def test_c2_pagerank_permutation_bit_exact(ref, tg, ctx, c2):
    off, tgt, tid = c2
    assert len(tgt) == 47_262_823  # R-MAT after rejection + dedup
    g = tg.CsrGraph(off, tgt)
    got = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(tid), ctx=ctx)
    want = ref.weighted_reverse_pagerank(off, tgt, tid)
    assert got.tobytes() == want.tobytes()
    perm = tg.permutation_from_scores(got, ctx=ctx)
    assert np.array_equal(perm.new_id_of, ref.permutation_from_scores(want))


def test_c2_reorder_sample_gather(ref, tg, ctx, c2):
    from paper_2111_05894_b200 import producers, synth
    off, tgt, tid = c2
    g = tg.CsrGraph(off, tgt)
    scores = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(tid), ctx=ctx)
    perm = tg.permutation_from_scores(scores, ctx=ctx)
    rg = tg.reorder_graph(g, perm, ctx=ctx)
    r_off, r_tgt = ref.reorder_graph(off, tgt, perm.new_id_of)
    assert np.array_equal(rg.offsets, r_off) and np.array_equal(rg.targets, r_tgt)
    gt = tg.transpose(rg, ctx=ctx)
    t_off, t_tgt = ref.transpose(r_off, r_tgt)
    assert np.array_equal(gt.offsets, t_off) and np.array_equal(gt.targets, t_tgt)
    del r_off, r_tgt

    new_tid = np.sort(perm.new_id_of[tid])
    fan, B = [15, 10, 5], 1024
    want_lists = ref.epoch_minibatches(t_off, t_tgt, new_tid, fan, B, 7, 0, max_batches=3)
    sampler = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(new_tid, 7, 0)
    got_lists = sampler.batches(order, fan, B, 7, 0, 0, 3)
    assert len(got_lists) == 3
    for a, b in zip(got_lists, want_lists):
        assert np.array_equal(a, b)

    feat = synth.test_features(N, DIM)
    lay = tg.plan_layout(N, 0.2, 0.0, 1, DIM, 4)
    store = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx)
    R = DIM * 4
    rf = oracle.RefFeatures(ref, feat.view(np.uint8).reshape(N, R)).reordered(perm.new_id_of)
    for ids in want_lists:
        rep = tg.TrafficReport()
        got = store.gather_rows(ids, report=rep)
        out = np.empty((len(ids), R), np.uint8)
        r6 = np.zeros(6, np.uint64)
        rf.gather(ref.plan_layout(N, 0.2, 0.0, 1, DIM, 4), ids, 0, out, r6)
        assert np.array_equal(got, out)
        assert np.array_equal(rep.as_array(), r6)
        assert 0 < rep.host_accesses < len(ids)  # both tiers exercised
