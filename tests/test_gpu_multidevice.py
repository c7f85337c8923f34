"""Partitioned PageRank over several devices of one process (tg_mgraph,
SURVEY §8e), run with VIRTUAL devices (several contexts on the one GPU this
build can use): the same code path as G physical GPUs, with same-device peer
copies. Bit-exact (raw bytes) against the reference for every device count,
like the reference's worker-count invariance (parallel.hpp:5-7)."""
import numpy as np
import pytest

import oracle
from tests.helpers import random_graph

pytestmark = pytest.mark.gpu


def checker():
    return oracle.ref() or oracle.port()


def _hub_graph(n, hubs, seed):
    rng = np.random.default_rng(seed)
    src = [rng.integers(0, n, 6 * n)]
    dst = [rng.integers(0, n, 6 * n)]
    for h, length in hubs:
        src.append(np.full(length, h))
        dst.append(rng.choice(n, size=length, replace=False))
    return oracle.port().from_edge_list(n, np.concatenate(src).astype(np.uint64),
                                        np.concatenate(dst).astype(np.uint64))


@pytest.fixture(scope="module")
def ctxs(tg, ctx):
    return [tg.Context(ctx.device) for _ in range(5)]


@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_mgraph_bit_exact_any_device_count(tg, ctxs, G):
    chk, port = checker(), oracle.port()
    cases = [random_graph(port, 400, 3.0, 2), _hub_graph(30000, [(0, 20000), (17, 5000),
                                                                  (29999, 3000)], 5)]
    for off, tgt in cases:
        n = len(off) - 1
        g = tg.CsrGraph(off, tgt)
        m = tg.MultiDeviceGraph(g, ctxs[:G])
        info = m.info()
        b = info["bounds"]
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b.astype(np.int64)) >= 0)
        assert np.array_equal(info["edges"], np.diff(off[b.astype(np.int64)]))
        assert np.array_equal(m.in_degrees(), port.in_degrees(off, tgt))  # sharded K1, summed
        tid = port.draw_random_train_ids(n, max(1, n // 10), 3)
        for it in (1, 5):
            got = m.weighted_reverse_pagerank(tg.PagerankConfig(it, 0.85), tg.TrainIdSet(tid))
            assert got.tobytes() == chk.weighted_reverse_pagerank(off, tgt, tid, it, 0.85).tobytes()
        got = m.reverse_pagerank(tg.PagerankConfig(3, 0.5))
        assert got.tobytes() == chk.reverse_pagerank(off, tgt, 3, 0.5).tobytes()
        with pytest.raises(tg.DomainError, match="out of range"):
            m.weighted_reverse_pagerank(tg.PagerankConfig(), tg.TrainIdSet(np.array([n], np.uint64)))
        with pytest.raises(tg.DomainError):
            m.weighted_reverse_pagerank(tg.PagerankConfig(), tg.TrainIdSet(np.zeros(0, np.uint64)))
        m.close()


def test_edge_balanced_blocks_on_rmat(tg):
    """Edge-balanced blocks on R-MAT (C1 shape): the largest block holds at
    most 1.1x the mean edge count at G = 2, 4, 8 (equal-row blocks: 3.4x at
    G = 8)."""
    from paper_2111_05894_b200 import synth
    off, tgt = synth.rmat_graph(1_000_000, 16_000_000, seed=1)
    e = len(tgt)
    for G in (2, 4, 8):
        b = tg.row_blocks(off, G).astype(np.int64)
        per = np.diff(off[b].astype(np.int64))
        assert per.sum() == e and per.max() <= 1.1 * e / G


def test_row_block_graph_contract(tg, ctx):
    """A row-block graph: steps only inside its block, whole-graph calls are
    DomainErrors, partial in-degrees sum to the whole."""
    import ctypes as C
    import torch
    from paper_2111_05894_b200._lib import LIB
    port = oracle.port()
    off, tgt = _hub_graph(5000, [(3, 3000)], 11)
    n = 5000
    bounds = [0, 1200, 3100, n]
    dev = torch.device("cuda", ctx.device)
    parts = []
    tot = torch.zeros(n, dtype=torch.int32, device=dev)
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        h = C.c_void_p()
        assert LIB.tg_graph_create_rows(ctx.h, off.ctypes.data, tgt.ctypes.data, n, len(tgt), r0, r1,
                                        C.byref(h)) == 0
        a, b = C.c_uint64(), C.c_uint64()
        assert LIB.tg_graph_row_range(h, C.byref(a), C.byref(b)) == 0 and (a.value, b.value) == (r0, r1)
        d = torch.empty(n, dtype=torch.int32, device=dev)
        assert LIB.tg_in_degrees_u32_async(ctx.h, h, d.data_ptr()) == 0
        ctx.sync()
        tot += d
        parts.append(h)
    assert np.array_equal(tot.cpu().numpy().astype(np.uint64), port.in_degrees(off, tgt))
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    out = np.empty(n, np.float64)
    h = parts[1]
    assert LIB.tg_reverse_pagerank(ctx.h, h, 5, 0.85, out.ctypes.data) == 2
    assert "rows" in LIB.tg_last_error().decode()
    assert LIB.tg_pagerank_step_async(ctx.h, h, tot.data_ptr(), 0.85, x.data_ptr(), x.data_ptr(),
                                      x.data_ptr(), 0, 100, 0) == 2  # rows outside the block
    assert LIB.tg_degree_score(ctx.h, h, out.ctypes.data) == 2
    assert LIB.tg_graph_offsets32(h) is None
    for h in parts:
        LIB.tg_graph_destroy(h)
