"""GPU minibatch expansion (csrc/sampling.cu) is bit-identical
to the reference's build_minibatch (sampling.cpp:56-90) and epoch schedule
(sampling.cpp:106-123). The checker is the reference build (oracle/_ref)
when present, else the pinned C restatement."""
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
    for h, length in hubs:  # nodes with many in-neighbours
        src.append(rng.choice(n, size=length, replace=False))
        dst.append(np.full(length, h))
    return port.from_edge_list(n, np.concatenate(src).astype(np.uint64),
                               np.concatenate(dst).astype(np.uint64))


@pytest.mark.parametrize("fanouts", [[10, 15], [15, 10, 5], [100, 3], [1], [2, 2, 2, 2, 2]])
def test_epoch_minibatches_bit_exact(tg, ctx, fanouts):
    from paper_2111_05894_b200 import producers
    chk = checker()
    n = 6000
    off, tgt = _graph(n, len(fanouts), hubs=[(0, 3000), (7, 500), (11, 65)])
    go, gt = chk.transpose(off, tgt)
    tid = oracle.port().draw_random_train_ids(n, 900, 3)
    want = chk.epoch_minibatches(go, gt, tid, fanouts, 64, 7, 1, max_batches=12)
    order = producers.epoch_order(tid, 7, 1)
    s = producers.GpuSampler(tg.CsrGraph(go, gt), ctx=ctx)
    for b, w in enumerate(want):
        got = s.minibatch(order[b * 64:(b + 1) * 64], fanouts, 7, 1, b)
        assert np.array_equal(got, w), f"batch {b}"


def test_build_minibatch_seeds_and_errors(tg, ctx):
    from paper_2111_05894_b200 import producers
    chk = checker()
    n = 500
    off, tgt = _graph(n, 5)
    go, gt = chk.transpose(off, tgt)
    s = producers.GpuSampler(tg.CsrGraph(go, gt), ctx=ctx)
    seeds = np.array([5, 3, 5, 499, 3], np.uint64)  # duplicates are fine (sampling.cpp:64-66)
    assert np.array_equal(s.minibatch(seeds, [4, 4], 1, 2, 3),
                          chk.build_minibatch(go, gt, seeds, [4, 4], 1, 2, 3))
    with pytest.raises(tg.DomainError, match="out of range"):
        s.minibatch(np.array([1, n], np.uint64), [3], 0, 0, 0)
    with pytest.raises(tg.DomainError):
        s.minibatch(np.array([1], np.uint64), [], 0, 0, 0)
    with pytest.raises(tg.DomainError):
        s.minibatch(np.array([1], np.uint64), [1, 1, 1, 1, 1, 1], 0, 0, 0)
    with pytest.raises(tg.DomainError):
        s.minibatch(np.array([1], np.uint64), [0], 0, 0, 0)
    with pytest.raises(tg.DomainError):
        s.minibatch(np.zeros(0, np.uint64), [3], 0, 0, 0)


def test_rmat_c1_shape_minibatches(tg, ctx):
    """C1 shape: the reference's (10, 15) fanout over the reordered R-MAT graph."""
    from paper_2111_05894_b200 import producers, synth
    chk = checker()
    off, tgt = synth.rmat_graph(200_000, 3_200_000, seed=1)
    n = len(off) - 1
    tid = oracle.port().draw_random_train_ids(n, n // 10, 3)
    go, gt = chk.transpose(off, tgt)
    want = chk.epoch_minibatches(go, gt, tid, [10, 15], 1024, 7, 0, max_batches=6)
    order = producers.epoch_order(tid, 7, 0)
    s = producers.GpuSampler(tg.CsrGraph(go, gt), ctx=ctx)
    for b, w in enumerate(want):
        assert np.array_equal(s.minibatch(order[b * 1024:(b + 1) * 1024], [10, 15], 7, 0, b), w)


@pytest.mark.parametrize("dedup", [True, False])
def test_training_trace_counts_bit_exact(tg, ctx, dedup):
    """run_training_trace (sampling.cpp:92-140) on the GPU: identical per-node
    access counts, with and without per-batch de-duplication, over 2 epochs."""
    from paper_2111_05894_b200 import producers
    ref = oracle.ref()
    if ref is None:
        pytest.skip("needs the reference build for run_training_trace")
    n = 4000
    off, tgt = _graph(n, 11, hubs=[(0, 2000), (3, 70)])
    go, gt = ref.transpose(off, tgt)
    tid = oracle.port().draw_random_train_ids(n, 700, 5)
    want = ref.run_training_trace(off, tgt, tid, [5, 10, 3], 50, 2, 9, dedup)
    s = producers.GpuSampler(tg.CsrGraph(go, gt), ctx=ctx)
    got = s.trace(tid, [5, 10, 3], 50, 2, 9, dedup)
    assert np.array_equal(got, want)


def test_raw_draws_multiset(tg, ctx):
    """raw_draws: each seed once as given plus every draw — its multiset summed
    over an epoch equals the reference's raw-access trace counts."""
    from paper_2111_05894_b200 import producers
    ref = oracle.ref()
    if ref is None:
        pytest.skip("needs the reference build for run_training_trace")
    n = 3000
    off, tgt = _graph(n, 12, hubs=[(1, 1500)])
    go, gt = ref.transpose(off, tgt)
    tid = oracle.port().draw_random_train_ids(n, 300, 6)
    want = ref.run_training_trace(off, tgt, tid, [4, 7], 64, 1, 3, False)
    s = producers.GpuSampler(tg.CsrGraph(go, gt), ctx=ctx)
    order = producers.epoch_order(tid, 3, 0)
    counts = np.zeros(n, np.uint64)
    for b in range((len(order) + 63) // 64):
        mem, raw = s.minibatch_raw(order[b * 64:(b + 1) * 64], [4, 7], 3, 0, b)
        assert np.array_equal(mem, np.unique(raw))
        np.add.at(counts, raw.astype(np.int64), np.uint64(1))
    assert np.array_equal(counts, want)


@pytest.mark.parametrize("lanes", ["1", "3", None, "7"])
@pytest.mark.parametrize("fanouts", [[10, 15], [15, 10, 5], [100, 3]])
def test_sample_batches_back_to_back(tg, ctx, monkeypatch, fanouts, lanes):
    """tg_sample_batches (one host round trip for many minibatches) gives the
    reference's epoch lists, from any first batch, incl. a short last batch,
    with any number of concurrent sampler lanes (TIERGRAPH_SAMPLER_LANES;
    default 4): batch k expands on lane k % L, compactions stay in order."""
    from paper_2111_05894_b200 import producers
    if lanes is not None:
        monkeypatch.setenv("TIERGRAPH_SAMPLER_LANES", lanes)
    chk = checker()
    n = 6000
    off, tgt = _graph(n, 7, hubs=[(0, 3000), (9, 400)])
    go, gt = chk.transpose(off, tgt)
    tid = oracle.port().draw_random_train_ids(n, 1000, 5)  # 16 batches of 64, the last 40
    want = chk.epoch_minibatches(go, gt, tid, fanouts, 64, 11, 2, max_batches=16)
    order = producers.epoch_order(tid, 11, 2)
    s = producers.GpuSampler(tg.CsrGraph(go, gt), ctx=ctx)
    got = s.batches(order, fanouts, 64, 11, 2)
    assert len(got) == 16 and all(np.array_equal(a, b) for a, b in zip(got, want))
    mid = s.batches(order, fanouts, 64, 11, 2, first_batch=5, nbatches=4)
    assert all(np.array_equal(a, b) for a, b in zip(mid, want[5:9]))
    md, offs = s.batches(order, fanouts, 64, 11, 2, device=True)  # left in HBM
    allm = md[:int(offs[-1])].cpu().numpy().view(np.uint64)
    assert all(np.array_equal(allm[int(offs[k]):int(offs[k + 1])], want[k]) for k in range(16))
    with pytest.raises(tg.DomainError, match="exceed"):
        s.batches(order, fanouts, 64, 11, 2, first_batch=15, nbatches=2)
