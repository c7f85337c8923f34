"""GPU parity: tier accounting, trace replays and the byte-moving tiered
gather (K7 placement + K8). Rows must be bit-exact: gathered row i ==
reorder_features(f, perm).row(ids[i]) (reorder.cpp:97-117 composed with
resolve tiering.cpp:48-65), and every TrafficReport must equal the
reference's gather() (tiering.cpp:100-125) integer for integer.
"""
import numpy as np
import pytest

import oracle
from tests.helpers import (RngStream, derive_stream_key, random_counter, random_graph,
                           random_layout, random_permutation)

pytestmark = pytest.mark.gpu

LISTING = (16, 4, 10, 2, 8, 4)


def checker():
    return oracle.ref() or oracle.port()


def test_account_known_answers(tg, ctx):  # test_tiering.cpp:124-153
    lay = tg.TierLayout(*LISTING)
    r = tg.TrafficReport()
    tg.gather(lay, [0, 1, 3], 0, r)
    assert r.host_bytes == 0 and r.local_accesses == 3 and r.local_bytes == 96
    cold = tg.TierLayout(16, 0, 0, 2, 8, 4)
    r = tg.TrafficReport()
    tg.gather(cold, [0, 5, 11, 15], 1, r)
    assert r.host_accesses == 4 and r.host_bytes == 128 and r.local_accesses + r.peer_accesses == 0
    r = tg.TrafficReport()
    tg.gather(lay, [2, 5, 11], 0, r)
    assert (r.local_accesses, r.peer_accesses, r.host_accesses) == (1, 1, 1)
    r = tg.TrafficReport()
    tg.gather(lay, [5], 1, r)
    assert r.local_accesses == 1


def test_account_errors_keep_prefix(tg, ctx):
    lay = tg.TierLayout(*LISTING)
    ids = [1, 5, 11, 16, 2]
    r = tg.TrafficReport(local_accesses=10)
    with pytest.raises(tg.DomainError, match="row 16 out of range for 16 rows"):
        tg.gather(lay, ids, 0, r)
    want = oracle.port().gather(LISTING, ids[:3], 0, np.array([10, 0, 0, 0, 0, 0], np.uint64))
    assert np.array_equal(r.as_array(), want)
    with pytest.raises(tg.DomainError, match="requesting device 2"):
        tg.gather(lay, [0], 2, tg.TrafficReport())
    tg.gather(lay, [], 7, tg.TrafficReport())  # empty: the reference loop never resolves


def test_account_random_layouts(tg, ctx):
    chk = checker()
    for i in range(40):
        rng = RngStream(derive_stream_key(i, [0xACC7]))
        n = 1 + rng.next_below(3000)
        lay = random_layout(rng, n)
        ids = np.random.default_rng(i).integers(0, n, 5000).astype(np.uint64)
        for dev in range(lay[3]):
            r = tg.TrafficReport()
            tg.gather(tg.TierLayout(*lay), ids, dev, r)
            assert np.array_equal(r.as_array(), chk.gather(lay, ids, dev))


def test_simulate_and_sweep(tg, ctx):
    chk = checker()
    for i in range(30):  # acceptance.cpp:384-411
        rng = RngStream(derive_stream_key(i, [0xB4]))
        n = 1 + rng.next_below(2000)
        lay = random_layout(rng, n)
        counts = random_counter(n, i + 900, tag=0x636E, bound=25)
        r = tg.simulate_trace(tg.make_access_counter(counts), tg.TierLayout(*lay))
        assert np.array_equal(r.as_array(), chk.simulate_trace(counts, lay))
        ordering = chk.score_ordering(counts.astype(np.float64))
        assert np.array_equal(tg.counts_in_row_order(tg.make_access_counter(counts), ordering),
                              chk.counts_in_row_order(counts, ordering))
        fr = [0.0, 0.05, 0.1, 0.25, 0.5, 1.0]
        rows = tg.hot_fraction_sweep(tg.make_access_counter(counts), ordering, fr, 0.1, lay[3], 8, 4)
        lays, reps, rf = chk.hot_fraction_sweep(counts, ordering, fr, 0.1, lay[3], 8, 4)
        for k, row in enumerate(rows):
            assert row.layout.as_tuple() == tuple(int(x) for x in lays[k])
            assert np.array_equal(row.report.as_array(), reps[k])
            assert row.replicated_fraction == rf[k]
    with pytest.raises(tg.DomainError):
        tg.simulate_trace(tg.make_access_counter([0, 0]), tg.TierLayout(2, 0, 1, 1, 1, 4))
    with pytest.raises(tg.DomainError):
        tg.simulate_trace(tg.make_access_counter([1, 1, 1]), tg.TierLayout(2, 0, 1, 1, 1, 4))
    c = tg.make_access_counter([9, 1, 4, 0, 2, 7, 3, 3, 1, 5])
    o = tg.score_ordering(c.counts.astype(np.float64))
    with pytest.raises(tg.DomainError):
        tg.hot_fraction_sweep(c, o, [0.5, 0.1], 0.0, 2, 4, 4)
    with pytest.raises(tg.DomainError, match="ordering"):
        tg.counts_in_row_order(c, np.array([0, 1, 2, 3, 4, 5, 6, 7, 8, 99], np.uint64))


def _virtual_devices(tg, ctx, features, perm, lay, **kw):
    """D stores on ONE GPU wired to each other's HBM slices through the same
    peer-pointer table real NVLink peers use (tg_store_set_peer)."""
    D = lay.num_devices
    stores = [tg.TieredFeatureStore(features, perm, lay, d, ctx=ctx, place=False, **kw)
              for d in range(D)]
    for d in range(1, D):
        stores[d].share_cold(stores[0])
    for s in stores:
        s.place(features, perm)
    for s in stores:
        for d in range(D):
            if d != s.device_index:
                s.set_peer(d, stores[d].local_base)
    return stores


@pytest.mark.parametrize("dim,eb", [(100, 4), (128, 4), (768, 2), (9, 4), (3, 1), (1, 8), (2048, 4),
                                    (36, 4), (300, 4), (1100, 4)])
@pytest.mark.parametrize("cold_mode,pad,split", [("reordered", False, False), ("indirect", False, False),
                                                 ("reordered", True, False), ("reordered", True, True),
                                                 ("reordered", False, True)])
@pytest.mark.parametrize("mode", ["ldg", "bulk", "bulk+spread", "l2pf+spread", "bulk+spread+dynamic"])
def test_store_gather_bit_exact(tg, ctx, dim, eb, cold_mode, pad, split, mode):
    """Rows byte-exact vs reorder_features (reorder.cpp:97-117) and the report
    equal to gather() (tiering.cpp:100-125) for every cold-tier format: split
    cold rows (TG_COLD_SPLIT_TAIL: 400 B -> 384 host + 16 HBM, 144 -> 128+16,
    1200 -> 1152+48, 4400 -> 4352+48 on the looped LDG path) included."""
    chk, port = checker(), oracle.port()
    n = 3000
    rng = np.random.default_rng(dim * eb)
    feat = rng.integers(0, 256, (n, dim * eb), dtype=np.uint8)
    perm = random_permutation(n, dim)
    reordered = port.reorder_features(feat, perm)
    for D, hot, rep in ((1, 0.2, 0.0), (2, 0.3, 0.05), (3, 0.5, 0.1), (4, 1.0, 0.0),
                        (6, 0.37, 0.2), (2, 0.0, 0.0)):
        lay = tg.plan_layout(n, hot, rep, D, dim, eb)
        stores = _virtual_devices(tg, ctx, feat, perm, lay, cold_mode=cold_mode, pad128=pad,
                                  split_tail=split, gather_mode=mode)
        ids = np.sort(rng.choice(n, size=700, replace=False)).astype(np.uint64)
        ids = np.concatenate([ids, rng.integers(0, n, 50).astype(np.uint64)])  # duplicates too
        for d, s in enumerate(stores):
            rep_ = tg.TrafficReport()
            out = s.gather_rows(ids, report=rep_)
            assert np.array_equal(out, reordered[ids])
            assert np.array_equal(rep_.as_array(), chk.gather(lay.as_tuple(), ids, d))


@pytest.mark.parametrize("mode", ["bulk+spread+dynamic", "bulk+dynamic"])
def test_dynamic_claims_rearm_between_launches(tg, ctx, mode):
    """TG_GATHER_DYNAMIC: the store's claim counter is re-armed by the last
    CTA of every launch, so back-to-back gathers of different lengths (sync
    and stream-ordered) each copy every row exactly once."""
    import torch
    n, dim = 20000, 100
    rng = np.random.default_rng(5)
    feat = rng.integers(0, 256, (n, dim * 4), dtype=np.uint8)
    perm = random_permutation(n, 3)
    reordered = oracle.port().reorder_features(feat, perm)
    lay = tg.plan_layout(n, 0.2, 0.0, 1, dim, 4)
    st = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx, gather_mode=mode)
    chk = checker()
    for size in (1, 31, 5000, 19000, 700, 12000):
        ids = np.sort(rng.choice(n, size=size, replace=False)).astype(np.uint64)
        rep_ = tg.TrafficReport()
        out = st.gather_rows(ids, report=rep_)
        assert np.array_equal(out, reordered[ids])
        assert np.array_equal(rep_.as_array(), chk.gather(lay.as_tuple(), ids, 0))
    dev = torch.device("cuda", ctx.device)
    lists = [np.sort(rng.choice(n, size=s_, replace=False)).astype(np.uint64)
             for s_ in (9000, 300, 15000)]
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    for ids in lists:
        out = torch.empty((len(ids), dim * 4), dtype=torch.uint8, device=dev)
        st.gather_rows_async(torch.as_tensor(ids.astype(np.int64), device=dev), out, cnt, err)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), reordered[ids])


def test_store_errors_and_empty(tg, ctx):
    n, dim = 100, 16
    feat = np.arange(n * dim, dtype=np.float32).reshape(n, dim)
    perm = random_permutation(n, 1)
    lay = tg.plan_layout(n, 0.3, 0.1, 1, dim, 4)
    s = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx)
    r = tg.TrafficReport()
    assert s.gather_rows(np.zeros(0, np.uint64), report=r).shape == (0, 64)
    with pytest.raises(tg.DomainError, match="row 100 out of range"):
        s.gather_rows([3, 50, 100, 4], report=r)
    assert np.array_equal(r.as_array(), oracle.port().gather(lay.as_tuple(), [3, 50], 0))
    with pytest.raises(tg.DomainError):
        tg.TieredFeatureStore(feat, np.zeros(n, np.uint64), lay, ctx=ctx)  # not a bijection
    lay2 = tg.plan_layout(n, 0.5, 0.0, 2, dim, 4)
    s2 = tg.TieredFeatureStore(feat, perm, lay2, 0, ctx=ctx)
    with pytest.raises(tg.DomainError, match="peer slice of device 1"):
        s2.gather_rows([60])
    with pytest.raises(tg.DomainError):
        tg.TieredFeatureStore(feat, perm, lay2, 2, ctx=ctx)


def test_device_resident_inputs_and_async(tg, ctx):
    import torch
    n, dim = 5000, 100
    from paper_2111_05894_b200 import synth
    feat = synth.test_features(n, dim)
    perm = random_permutation(n, 9)
    lay = tg.plan_layout(n, 0.2, 0.0, 1, dim, 4)
    dev = torch.device("cuda", ctx.device)
    feat_d = torch.from_numpy(feat).to(dev)
    s = tg.TieredFeatureStore(feat_d.view(torch.uint8).reshape(-1), perm, lay, ctx=ctx)
    ids = torch.randint(0, n, (4096,), device=dev, dtype=torch.int64)
    out = torch.empty((4096, dim * 4), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    ctx.sync()
    s.gather_rows_async(ids, out, cnt, err)
    ctx.sync()
    inv = oracle.port().invert(perm)
    old = inv[ids.cpu().numpy().astype(np.uint64)]
    want = synth.expected_rows(old, dim)
    assert np.array_equal(out.cpu().numpy().view(np.float32), want)
    rep = oracle.port().gather(lay.as_tuple(), ids.cpu().numpy().astype(np.uint64), 0)
    assert cnt.cpu().tolist() == [int(rep[0]), int(rep[1]), int(rep[2])]
    assert int(err.item()) == -1


def test_end_to_end_reference_minibatches(tg, ctx):
    """The whole path on a small R-MAT graph: wrpr -> permutation -> reorder
    graph/features -> the reference's OWN sampled minibatch id lists ->
    tiered gather; rows byte-equal and reports equal to the reference."""
    chk = checker()
    if chk.kind != "reference":
        pytest.skip("needs the reference build for its minibatch lists")
    from paper_2111_05894_b200 import producers, synth
    n, dim = 50_000, 128
    off, tgt = synth.rmat_graph(n, 800_000, seed=1)
    tid = chk.draw_random_train_ids(n, n // 10, 3)
    scores = tg.weighted_reverse_pagerank(tg.CsrGraph(off, tgt), tg.PagerankConfig(),
                                          tg.TrainIdSet(tid))
    assert scores.tobytes() == chk.weighted_reverse_pagerank(off, tgt, tid).tobytes()
    perm = tg.permutation_from_scores(scores)
    assert np.array_equal(perm.new_id_of, chk.permutation_from_scores(scores))
    rg = tg.reorder_graph(tg.CsrGraph(off, tgt), perm)
    ro, rt = chk.reorder_graph(off, tgt, perm.new_id_of)
    assert np.array_equal(rg.offsets, ro) and np.array_equal(rg.targets, rt)
    go, gt = chk.transpose(ro, rt)
    new_tid = np.sort(perm.new_id_of[tid])
    lists = chk.epoch_minibatches(go, gt, new_tid, [10, 15], 1024, 7, 0, max_batches=4)
    mine = producers.epoch_minibatches(tg.CsrGraph(go, gt), new_tid, [10, 15], 1024, 7, 0,
                                       max_batches=4)
    assert all(np.array_equal(a, b) for a, b in zip(lists, mine))
    feat = chk.make_test_features(n, dim)
    reordered = chk.reorder_features(feat, perm.new_id_of)
    lay = tg.plan_layout(n, 0.2, 0.0, 1, dim, 4)
    store = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx)
    for ids in lists:
        r = tg.TrafficReport()
        out = store.gather_rows(ids, report=r)
        assert np.array_equal(out.view(np.float32), reordered[ids])
        assert np.array_equal(r.as_array(), chk.gather(lay.as_tuple(), ids, 0))


@pytest.mark.parametrize("cold_mode", ["indirect", "reordered"])
def test_place_rows_from_a_row_cache(tg, ctx, cold_mode):
    """tg_store_place_rows: new id i holds rows[row_of[i]] (the C4 row-cache
    placement); with row_of = inverse permutation it is tg_store_place."""
    chk = checker()
    n, dim, P = 5000, 24, 1237
    rng = np.random.default_rng(5)
    perm = rng.permutation(n).astype(np.uint64)
    inv = np.empty(n, np.uint64)
    inv[perm.astype(np.int64)] = np.arange(n, dtype=np.uint64)
    rows = rng.integers(0, 256, (P, dim * 2), dtype=np.uint8)
    row_of = (inv % np.uint64(P)).astype(np.uint32)
    lay = tg.plan_layout(n, 0.3, 0.1, 1, dim, 2)
    st = tg.TieredFeatureStore(None, tg.NodePermutation(perm), lay, ctx=ctx, cold_mode=cold_mode,
                               place=False)
    st.place_rows(rows, row_of)
    ids = np.unique(rng.integers(0, n, 3000)).astype(np.uint64)
    rep = tg.TrafficReport()
    out = st.gather_rows(ids, report=rep)
    assert np.array_equal(out.reshape(len(ids), -1), rows[row_of[ids.astype(np.int64)]])
    assert np.array_equal(rep.as_array(), chk.gather(lay.as_tuple(), ids, 0))
    # the identity map over the original matrix is tg_store_place
    feat = rng.integers(0, 256, (n, dim * 2), dtype=np.uint8)
    st2 = tg.TieredFeatureStore(feat, tg.NodePermutation(perm), lay, ctx=ctx, cold_mode=cold_mode)
    st.place_rows(feat, inv.astype(np.uint32))
    assert np.array_equal(st.gather_rows(ids), st2.gather_rows(ids))
    with pytest.raises(tg.DomainError, match="row_of"):
        st.place_rows(rows, np.full(n, P, np.uint32))
    # the cold part timed alone (measurement helper) runs on the placed store
    assert st.measure_cold_us(100, 2) > 0


def test_time_gather_rows_matches_gather_rows(tg, ctx):
    """tg_time_gather_rows (the bench's e2e timer) runs the public
    tg_gather_rows per list: same bytes, same accumulated report."""
    chk = checker()
    n, dim = 4000, 32
    rng = np.random.default_rng(9)
    perm = rng.permutation(n).astype(np.uint64)
    feat = rng.integers(0, 256, (n, dim * 4), dtype=np.uint8)
    lay = tg.plan_layout(n, 0.25, 0.0, 1, dim, 4)
    st = tg.TieredFeatureStore(feat, tg.NodePermutation(perm), lay, ctx=ctx)
    lists = [np.unique(rng.integers(0, n, 700)).astype(np.uint64) for _ in range(4)]
    out = np.zeros((max(len(x) for x in lists), dim * 4), np.uint8)
    rep = tg.TrafficReport()
    sec = st.time_gather_rows(lists, out, rep)
    assert sec > 0
    want = np.zeros(6, np.uint64)
    for x in lists:
        want = chk.gather(lay.as_tuple(), x, 0, want)
    assert np.array_equal(rep.as_array(), want)
    assert np.array_equal(out[:len(lists[-1])], st.gather_rows(lists[-1]))
