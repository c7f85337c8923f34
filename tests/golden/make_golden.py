"""Generates tests/golden/golden_small.npz from the UNMODIFIED reference build
(oracle/_ref/libtgref.so, compiled from /root/reference by oracle/Makefile).

Run here, where /root/reference exists:  python tests/golden/make_golden.py
The fixture then travels with the repo, so the GPU tests and the CPU port are
pinned to the reference's own outputs even where the reference is absent.

Everything comes from reference calls:
  graph      generate_power_law(n, m, seed) (csr_graph.cpp:95-132, BA model)
  train ids  draw_random_train_ids (scoring.cpp:22-31)
  in-degrees in_degrees (csr_graph.cpp:89-93)
  scores     weighted_reverse_pagerank (scoring.cpp:86-102), 5 iterations, d = 0.85
  perm       permutation_from_scores (reorder.cpp:23-29)
  graph'     reorder_graph (reorder.cpp:39-66) and its transpose (csr_graph.cpp:67-80)
  lists      the epoch's first minibatches (sampling.cpp:56-90, 106-123)
  layouts    plan_layout (tiering.cpp:67-98); reports gather (tiering.cpp:100-125)
  rows       sha256 of reorder_features(make_test_features)[ids] (reorder.cpp:97-117)
  sweep      hot_fraction_sweep of the lists' access counts (tiering.cpp:177-202)
  graph 2    hub rows of 6000 / 2500 / 700 edges (every K3 row class), its
             weighted and plain (7 iterations, d = 0.5) scores and permutation
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

N, M, SEED = 3000, 4, 1
TRAIN, DIM = 300, 16
FANOUTS, BATCH, NB = (10, 15), 64, 3
LAYOUTS = [(0.2, 0.0, 1), (0.3, 0.05, 2), (0.5, 0.1, 3)]
FRACTIONS = [0.0, 0.1, 0.2, 0.5, 1.0]


def main():
    import oracle
    ref = oracle.ref()
    if ref is None:
        raise SystemExit("oracle/_ref is not built (needs /root/reference): run `make -C oracle`")
    off, tgt = ref.generate_power_law(N, M, SEED)
    tid = ref.draw_random_train_ids(N, TRAIN, 3)
    indeg = ref.in_degrees(off, tgt)
    scores = ref.weighted_reverse_pagerank(off, tgt, tid)
    perm = ref.permutation_from_scores(scores)
    roff, rtgt = ref.reorder_graph(off, tgt, perm)
    goff, gtgt = ref.transpose(roff, rtgt)
    new_tid = np.sort(perm[tid])
    lists = ref.epoch_minibatches(goff, gtgt, new_tid, list(FANOUTS), BATCH, 7, 0, max_batches=NB)
    feat = ref.make_test_features(N, DIM)
    reordered = ref.reorder_features(feat, perm)
    out = dict(off=off, tgt=tgt, tid=tid, indeg=indeg, scores=scores, perm=perm,
               goff=goff, gtgt=gtgt, fanouts=np.array(FANOUTS, np.uint32),
               params=np.array([N, M, SEED, TRAIN, DIM, BATCH, NB], np.uint64))
    lens = np.array([len(x) for x in lists], np.uint64)
    out["list_lens"] = lens
    out["lists"] = np.concatenate(lists).astype(np.uint64)
    rows = []
    for x in lists:
        rows.append(np.frombuffer(hashlib.sha256(np.ascontiguousarray(reordered[x.astype(np.int64)])
                                                 .tobytes()).digest(), np.uint8))
    out["rows_sha256"] = np.stack(rows)
    lays, reps = [], []
    for hot, rep, d in LAYOUTS:
        lay = ref.plan_layout(N, hot, rep, d, DIM, 4)
        lays.append(lay)
        for x in lists:
            for dev in range(d):
                reps.append(ref.gather(lay, x, dev))
    out["layouts"] = np.array(lays, np.uint64)
    out["reports"] = np.array(reps, np.uint64)
    counts = np.zeros(N, np.uint64)
    for x in lists:
        np.add.at(counts, x.astype(np.int64), np.uint64(1))
    order = np.argsort(perm, kind="stable").astype(np.uint64)  # new id -> old id
    counts_old = np.zeros(N, np.uint64)
    counts_old[order.astype(np.int64)] = counts
    sl, sr, sf = ref.hot_fraction_sweep(counts_old, order, FRACTIONS, 0.05, 2, DIM, 4)
    out.update(counts_old=counts_old, order=order, fractions=np.array(FRACTIONS),
               sweep_layouts=sl, sweep_reports=sr, sweep_rep=sf)
    # a second graph with long rows (K3 classes A, B and C): hub rows 0..2
    # with 6000 / 2500 / 700 out-edges plus random edges, canonicalised by the
    # reference's from_edge_list (csr_graph.cpp:36-65)
    rng = np.random.default_rng(11)
    n2 = 8000
    src = [np.zeros(6000, np.uint64), np.ones(2500, np.uint64), np.full(700, 2, np.uint64),
           rng.integers(0, n2, 40000).astype(np.uint64)]
    dst = [rng.choice(n2, 6000, replace=False).astype(np.uint64),
           rng.choice(n2, 2500, replace=False).astype(np.uint64),
           rng.choice(n2, 700, replace=False).astype(np.uint64),
           rng.integers(0, n2, 40000).astype(np.uint64)]
    off2, tgt2 = ref.from_edge_list(n2, np.concatenate(src), np.concatenate(dst))
    tid2 = ref.draw_random_train_ids(n2, 800, 5)
    out.update(off2=off2, tgt2=tgt2, tid2=tid2,
               scores2=ref.weighted_reverse_pagerank(off2, tgt2, tid2),
               scores2_plain=ref.reverse_pagerank(off2, tgt2, 7, 0.5))
    out["perm2"] = ref.permutation_from_scores(out["scores2"])
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    print(f"golden_small.npz: {N} nodes / {len(tgt)} edges, {len(lists)} minibatches "
          f"({', '.join(str(len(x)) for x in lists)} ids), {len(reps)} reports")


if __name__ == "__main__":
    main()
