"""GPU parity: transpose (csr_graph.cpp:67-80) on the device is identical to
the reference: every transposed row lists its sources in ascending order,
duplicates and empty rows included."""
import numpy as np
import pytest

import oracle
from paper_2111_05894_b200 import synth
from tests.helpers import random_graph

pytestmark = pytest.mark.gpu


def checker():
    return oracle.ref() or oracle.port()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_transpose_random_graphs(tg, ctx, seed):
    chk = checker()
    port = oracle.port()
    off, tgt = random_graph(port, 700 + 300 * seed, 6.0, seed)
    t_off, t_tgt = chk.transpose(off, tgt)
    g = tg.transpose(tg.CsrGraph(off, tgt), ctx=ctx)
    assert np.array_equal(g.offsets, t_off) and np.array_equal(g.targets, t_tgt)


def test_transpose_non_canonical_and_edge_cases(tg, ctx):
    chk = checker()
    # duplicate edges, unsorted rows, empty first / last rows, a self loop
    off = np.array([0, 0, 4, 4, 7, 7], np.uint64)
    tgt = np.array([3, 1, 3, 1, 0, 3, 3], np.uint64)
    t_off, t_tgt = chk.transpose(off, tgt)
    g = tg.transpose(tg.CsrGraph(off, tgt), ctx=ctx)
    assert np.array_equal(g.offsets, t_off) and np.array_equal(g.targets, t_tgt)
    # no edges
    g0 = tg.transpose(tg.CsrGraph(np.zeros(4, np.uint64), np.zeros(0, np.uint64)), ctx=ctx)
    assert np.array_equal(g0.offsets, np.zeros(4, np.uint64)) and g0.num_edges() == 0
    with pytest.raises(tg.FormatError):
        tg.transpose(tg.CsrGraph(np.array([0, 1], np.uint64), np.array([5], np.uint64)), ctx=ctx)


def test_transpose_rmat_c1_scale(tg, ctx):
    off, tgt = synth.rmat_graph(1_000_000, 16_000_000, seed=1)
    t_off, t_tgt = oracle.port().transpose(off, tgt)
    g = tg.transpose(tg.CsrGraph(off, tgt), ctx=ctx)
    assert np.array_equal(g.offsets, t_off) and np.array_equal(g.targets, t_tgt)
