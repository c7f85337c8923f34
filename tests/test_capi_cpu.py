"""CPU-side checks of the product library (no GPU needed).

* libtiergraph_b200.so loads and exports every symbol include/tg_capi.h declares;
* the host-scalar C-ABI (resolve / plan_layout / report helpers) agrees with
  the oracle on the reference tests' known answers and random layouts;
* the host producers (train ids, transpose, minibatch id lists) are
  bit-identical to the reference build.
"""
import os
import re

import numpy as np
import pytest

import oracle
from tests.helpers import RngStream, derive_stream_key, random_graph, random_layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "tg_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import subprocess
    so = os.path.join(ROOT, "paper_2111_05894_b200", "libtiergraph_b200.so")
    assert os.path.exists(so), "build the library first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (tg_[a-z0-9_]+)$", out, flags=re.M))
    declared = _declared_symbols()
    assert len(declared) > 50
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header():
    from paper_2111_05894_b200 import _lib
    assert sorted(_lib.SIGNATURES) == _declared_symbols()


def test_no_gpu_context_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2111_05894_b200 import tiergraph as tg
    with pytest.raises(tg.TierGraphError):
        tg.Context(0)


LISTING = (16, 4, 10, 2, 8, 4)


def test_resolve_and_layout_known_answers():
    from paper_2111_05894_b200 import tiergraph as tg
    lay = tg.TierLayout(*LISTING)
    assert tg.resolve(lay, 2, 0) == tg.Location(tg.Tier.LocalHot, 0, 2)
    assert tg.resolve(lay, 5, 0) == tg.Location(tg.Tier.InterleavedDevice, 1, 0)
    assert tg.resolve(lay, 11, 0) == tg.Location(tg.Tier.ColdHost, 0, 1)
    with pytest.raises(tg.DomainError):
        tg.resolve(lay, 16, 0)
    with pytest.raises(tg.DomainError):
        tg.resolve(lay, 0, 2)
    mid = tg.plan_layout(100, 0.10, 0.05, 4, 8, 4)
    assert (mid.local_boundary, mid.multi_boundary) == (5, 10)
    with pytest.raises(tg.DomainError, match="640"):
        tg.plan_layout(100, 0.5, 0.1, 4, 8, 4, 639)
    assert tg.plan_layout(100, 0.5, 0.1, 4, 8, 4, 640).multi_boundary == 50
    with pytest.raises(tg.DomainError):
        tg.plan_layout(100, 0.2, 0.5, 4, 8, 4)
    with pytest.raises(tg.DomainError):
        tg.validate_cost_model(tg.LinkCostModel(local_gbps=0.0))
    r = tg.TrafficReport(local_bytes=9_000_000_000, peer_bytes=1_500_000_000,
                         host_bytes=160_000_000)
    assert r.est_transfer_seconds(tg.LinkCostModel(0.9, 0.15, 0.016)) == pytest.approx(30.0)
    assert tg.TrafficReport(local_accesses=3, host_accesses=1).hit_ratio() == 0.75
    assert tg.TrafficReport().hit_ratio() == 0.0


def test_resolve_matches_oracle_on_random_layouts():
    from paper_2111_05894_b200 import tiergraph as tg
    port = oracle.port()
    for i in range(40):
        rng = RngStream(derive_stream_key(i, [0x8]))
        n = 1 + rng.next_below(500)
        lay = random_layout(rng, n)
        L = tg.TierLayout(*lay)
        for row in range(0, n, 3):
            for dev in range(lay[3]):
                got = tg.resolve(L, row, dev)
                assert (got.tier, got.device, got.row_within_tier) == port.resolve(lay, row, dev)
        for f in (0.0, 0.05, 0.33, 1.0):
            a = tg.plan_layout(n, f, f / 3, lay[3], lay[4], lay[5])
            assert a.as_tuple() == port.plan_layout(n, f, f / 3, lay[3], lay[4], lay[5])


def test_host_producers_match_reference(ref):
    from paper_2111_05894_b200 import producers, tiergraph as tg
    port = oracle.port()
    for seed in range(4):
        n = 300 + 97 * seed
        off, tgt = random_graph(port, n, 4.0, seed)
        tid = producers.draw_random_train_ids(n, n // 7, seed)
        assert np.array_equal(tid.ids, ref.draw_random_train_ids(n, n // 7, seed))
        gt = producers.transpose(tg.CsrGraph(off, tgt))
        go, gtt = ref.transpose(off, tgt)
        assert np.array_equal(gt.offsets, go) and np.array_equal(gt.targets, gtt)
        for fan, bs in (([10, 15], 16), ([15, 10, 5], 8), ([3], 50), ([70, 2], 7)):
            mine = producers.epoch_minibatches(gt, tid, fan, bs, seed=7, epoch=seed)
            theirs = ref.epoch_minibatches(go, gtt, tid.ids, fan, bs, 7, seed)
            assert len(mine) == len(theirs)
            for a, b in zip(mine, theirs):
                assert np.array_equal(a, b)
    with pytest.raises(tg.DomainError):
        producers.draw_random_train_ids(10, 11, 0)


def test_epoch_order_matches_reference_shuffle():
    """producers.epoch_order = the reference's per-epoch Fisher-Yates
    (sampling.cpp:106-109, rng.hpp:67-73), checked on the oracle."""
    import oracle
    from paper_2111_05894_b200 import producers
    port = oracle.port()
    chk = oracle.ref() or port
    tid = port.draw_random_train_ids(10_000, 1_234, 9)
    for epoch in (0, 1, 7):
        key = chk.derive_stream_key(7, [0x5348, epoch])
        assert np.array_equal(producers.epoch_order(tid, 7, epoch), port.shuffle(key, tid))
