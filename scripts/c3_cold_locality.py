"""Experiment: at C3 scale (papers100M-shaped, hot 20 %), how concentrated are
the cold-row accesses, and does a physical cold-tier order that packs the
likely-read rows into the first few GB (fewer host-page translation misses)
shorten K8? Orders compared (the cold tier read in place through a row map,
TG_COLD_INDIRECT + tg_store_place_rows; row CONTENTS are not checked here):

  newid   cold row r at position r (today's reordered tier)
  degree  cold rows by out-degree in the reordered graph (the in-neighbour
          sampler reaches u through every row of the transpose u appears in)
  seen    rows read by the first half of the epoch's minibatches first (by
          count, then new id), then the rest in new-id order

Timed on minibatches of the second half (not used to build any order).
Not part of the bench."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import producers, tiergraph as tg
    cfg = dict(bench.CONFIGS["c3"])
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = tg.Context(0, stream=s)
    off, tgt, tid = bench.build_inputs(cfg, 0)
    n = len(off) - 1
    g = tg.CsrGraph(off, tgt)
    scores = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tid, ctx=ctx)
    perm = tg.permutation_from_scores(scores, ctx=ctx)
    rg = tg.reorder_graph(g, perm, ctx=ctx)
    del g
    outdeg = np.diff(rg.offsets.astype(np.int64))
    gt = producers.transpose(rg)
    del rg
    new_tid = np.sort(perm.new_id_of[tid.ids])
    sampler = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(new_tid, 7, 0)
    lists = [sampler.minibatch(order[b * 1024:(b + 1) * 1024], cfg["fanouts"], 7, 0, b)
             for b in range(nb)]
    del sampler, gt
    lay = tg.plan_layout(n, 0.2, 0.0, 1, cfg["dim"], cfg["elem"])
    mb = lay.multi_boundary
    ncold = n - mb
    R = cfg["dim"] * cfg["elem"]
    half = nb // 2
    train = np.concatenate([x[x >= mb] for x in lists[:half]]) - mb
    evals = np.concatenate([x[x >= mb] for x in lists[half:]]) - mb
    print(f"cold rows {ncold}, cold accesses per minibatch {len(evals) / (nb - half):.0f}", flush=True)

    # physical position of every cold row under each order
    cold_ids = np.arange(ncold, dtype=np.int64)
    pos = {"newid": cold_ids}
    deg = outdeg[mb:]
    o = np.lexsort((cold_ids, -deg))
    p = np.empty(ncold, np.int64)
    p[o] = cold_ids
    pos["degree"] = p
    cnt = np.bincount(train.astype(np.int64), minlength=ncold)
    o = np.lexsort((cold_ids, -cnt))
    p = np.empty(ncold, np.int64)
    p[o] = cold_ids
    pos["seen"] = p
    print(f"rows seen in the first half: {np.count_nonzero(cnt)} "
          f"({np.count_nonzero(cnt) * R / 1e9:.2f} GB)", flush=True)
    gbs = [0.5, 1, 2, 4, 8, 16, 32]
    for name, p in pos.items():
        off_gb = p[evals.astype(np.int64)] * R / 1e9
        fr = [float(np.mean(off_gb < x)) for x in gbs]
        print(f"{name:7s} share of second-half cold reads within the first "
              + ", ".join(f"{x:g} GB: {f:.3f}" for x, f in zip(gbs, fr)), flush=True)

    feat, _, _ = bench.pin_features(cfg)
    dev = torch.device("cuda", 0)
    timed = lists[half:half + 60]
    ids_d = [torch.as_tensor(x.astype(np.int64), device=dev) for x in timed]
    maxu = max(len(x) for x in timed)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = torch.empty((maxu, R), dtype=torch.uint8, device=dev)
    cnt_d = torch.zeros(3, dtype=torch.int64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    for name in ["newid", "degree", "seen", "newid"]:
        row_of = np.arange(n, dtype=np.uint32)
        row_of[mb:] = (mb + pos[name]).astype(np.uint32)
        st = tg.TieredFeatureStore(None, perm, lay, ctx=ctx, cold_mode="indirect", place=False)
        st.place_rows(feat, row_of)
        for k in range(3):
            st.gather_rows_async(ids_d[k], out, cnt_d, err)
        ts = []
        for k in range(3, len(timed)):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            st.gather_rows_async(ids_d[k], out, cnt_d, err)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = np.array([a.elapsed_time(b) for a, b in ts])
        # the cold rows alone
        tc = []
        for k in range(3, len(timed)):
            cold = ids_d[k][ids_d[k] >= mb]
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            st.gather_rows_async(cold, out, cnt_d, err)
            b.record()
            tc.append((a, b))
        torch.cuda.synchronize()
        mc = np.array([a.elapsed_time(b) for a, b in tc])
        print(f"order {name:7s} K8 avg {ms.mean() * 1e3:7.1f} us (min {ms.min() * 1e3:6.1f})  "
              f"cold rows alone {mc.mean() * 1e3:7.1f} us", flush=True)
        st.close()


if __name__ == "__main__":
    main()
