"""GPU parity: the reference's binary containers loaded straight into the
device tiers. Files are WRITTEN BY THE REFERENCE
(io.cpp save_csr / save_features / save_u64_vector via oracle/_ref); the
device graph must give bit-identical PageRank and in-degrees, the placed
store byte-identical rows, and header errors the reference's exception class
and message (io.cpp:40-46, 65-75, 95-110, 163-180).
"""
import struct

import numpy as np
import pytest

import oracle
from paper_2111_05894_b200 import synth
from tests.helpers import random_graph, random_permutation

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def refo():
    r = oracle.ref()
    if r is None:
        pytest.skip("reference build oracle/_ref/libtgref.so not present")
    return r


def test_csrg_into_device_graph(tg, ctx, refo, tmp_path):
    off, tgt = synth.rmat_graph(60_000, 900_000, seed=4)
    path = tmp_path / "g.csrg"
    refo.save_csr(off, tgt, path)
    g = tg.load_csr_device(path, ctx=ctx)
    assert (g.num_nodes(), g.num_edges()) == (len(off) - 1, len(tgt))
    tid = refo.draw_random_train_ids(len(off) - 1, 6000, 3)
    got = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tg.TrainIdSet(tid), ctx=ctx)
    want = refo.weighted_reverse_pagerank(off, tgt, tid)
    assert got.tobytes() == want.tobytes()
    assert np.array_equal(tg.in_degrees(g, ctx=ctx), refo.in_degrees(off, tgt))
    # a chunk boundary inside offsets and targets (64 MB staging = 8M entries)
    off2, tgt2 = synth.rmat_graph(9_000_000, 9_500_000, seed=5)
    p2 = tmp_path / "g2.csrg"
    refo.save_csr(off2, tgt2, p2)
    g2 = tg.load_csr_device(p2, ctx=ctx)
    assert np.array_equal(tg.in_degrees(g2, ctx=ctx),
                          np.bincount(tgt2.astype(np.int64), minlength=len(off2) - 1))


def _expect_same_error(tg, refo_call, ours_call):
    with pytest.raises(Exception) as want:
        refo_call()
    with pytest.raises(Exception) as got:
        ours_call()
    assert type(got.value).__name__ == type(want.value).__name__
    assert str(got.value) == str(want.value)


def test_csrg_header_errors_match_reference(tg, ctx, refo, tmp_path):
    off = np.array([0, 2, 3, 3], np.uint64)
    tgt = np.array([1, 2, 0], np.uint64)
    good = tmp_path / "good.csrg"
    refo.save_csr(off, tgt, good)
    raw = good.read_bytes()
    cases = {
        "magic.csrg": b"GRSC" + raw[4:],
        "version.csrg": raw[:4] + struct.pack("<I", 7) + raw[8:],
        "trunc_head.csrg": raw[:10],
        "trunc_off.csrg": raw[:24 + 8 * 2],
        "trunc_tgt.csrg": raw[:-4],
    }
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        _expect_same_error(tg, lambda: refo.load_csr(p), lambda: tg.load_csr_device(p, ctx=ctx))
    missing = tmp_path / "missing.csrg"
    _expect_same_error(tg, lambda: refo.load_csr(missing), lambda: tg.load_csr_device(missing, ctx=ctx))
    # semantic validation (validate_csr) raises the same class
    bad = tmp_path / "range.csrg"
    bad.write_bytes(raw[:-8] + struct.pack("<Q", 9))
    with pytest.raises(tg.FormatError):
        tg.load_csr_device(bad, ctx=ctx)


@pytest.mark.parametrize("dim", [20, 100])
@pytest.mark.parametrize("D,rep,hot", [(1, 0.0, 0.25), (3, 0.1, 0.6)])
def test_feat_into_store(tg, ctx, refo, tmp_path, D, rep, hot, dim):
    n, eb = 3001, 4
    rng = np.random.default_rng(D)
    feat = rng.integers(0, 256, (n, dim * eb), dtype=np.uint8)
    path = tmp_path / "f.feat"
    refo.save_features(feat, n, dim, eb, path)
    perm = random_permutation(n, 11 + D)
    inv = np.empty(n, np.uint64)
    inv[perm.astype(np.int64)] = np.arange(n, dtype=np.uint64)
    lay = tg.plan_layout(n, hot, rep, D, dim, eb)
    ids = np.unique(rng.integers(0, n, 1500)).astype(np.uint64)
    for dev in range(D):
        st = tg.TieredFeatureStore(None, tg.NodePermutation(perm), lay, dev, ctx=ctx, place=False)
        st.place_file(path, perm)
        # rows another device owns are not in this store: gather the ones it serves
        if D > 1:
            peers = [tg.TieredFeatureStore(feat, tg.NodePermutation(perm), lay, d, ctx=ctx)
                     for d in range(D) if d != dev]
            for p_st, d in zip(peers, [d for d in range(D) if d != dev]):
                st.set_peer(d, p_st.local_base)
        rep_ = tg.TrafficReport()
        out = st.gather_rows(ids, report=rep_)
        assert np.array_equal(out, feat[inv[ids.astype(np.int64)].astype(np.int64)])
        assert np.array_equal(rep_.as_array(), refo.gather(lay.as_tuple(), ids, dev))


def test_feat_errors(tg, ctx, refo, tmp_path):
    n, dim, eb = 10, 3, 4
    feat = np.arange(n * dim * eb, dtype=np.uint8).reshape(n, dim * eb)
    good = tmp_path / "good.feat"
    refo.save_features(feat, n, dim, eb, good)
    raw = good.read_bytes()
    lay = tg.plan_layout(n, 0.5, 0.0, 1, dim, eb)
    perm = np.arange(n, dtype=np.uint64)
    cases = {
        "magic.feat": b"TAEF" + raw[4:],
        "version.feat": raw[:4] + struct.pack("<I", 2) + raw[8:],
        "trunc_head.feat": raw[:20],
        "trunc_data.feat": raw[:-5],
    }
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        want = refo.load_features_error(p)
        assert want is not None
        st = tg.TieredFeatureStore(None, perm, lay, ctx=ctx, place=False)
        with pytest.raises(tg.FormatError) as got:
            st.place_file(p, perm)
        assert want[0] == 3 and str(got.value) == want[1]
    st = tg.TieredFeatureStore(None, perm, tg.plan_layout(n, 0.5, 0.0, 1, dim + 1, eb), ctx=ctx,
                               place=False)
    with pytest.raises(tg.FormatError, match="layout has"):
        st.place_file(good, perm)
    st = tg.TieredFeatureStore(None, perm, lay, ctx=ctx, cold_mode="indirect", place=False)
    with pytest.raises(tg.DomainError, match="TG_COLD_INDIRECT"):
        st.place_file(good, perm)
    st = tg.TieredFeatureStore(None, perm, lay, ctx=ctx, place=False)
    with pytest.raises(tg.IoError):
        st.place_file(tmp_path / "missing.feat", perm)
    with pytest.raises(tg.DomainError, match="permutation"):
        st.place_file(good, np.zeros(n, np.uint64))
