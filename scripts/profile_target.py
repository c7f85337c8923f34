"""Short, self-contained targets for ncu at full config size (C3/C4).

ncu's kernel replay cannot save/restore K8's working set at C3 (45 GB of
mapped host memory; profiles/r01ai ncu_gather_c3.log), so K8 is profiled with
`--replay-mode application`, which re-runs the whole process once per pass.
That is only affordable if one pass is short, so the expensive inputs (the
permutation and the epoch's minibatch id lists, which need PageRank, the
selection, reorder_graph, transpose and the sampler) are made ONCE by `prep`
and cached under /tmp; `k8` then only fills the features and builds the store.

  python scripts/profile_target.py prep --config c3
  ncu --replay-mode application ... python scripts/profile_target.py k8 --config c3
  ncu -k regex:pr_step ...          python scripts/profile_target.py k3 --config c3
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (CONFIGS, fixtures)


def cache_path(config):
    return f"/tmp/tg_prof_{config}.npz"


def prep(args):
    import torch
    from paper_2111_05894_b200 import producers, tiergraph as tg
    cfg = bench.CONFIGS[args.config]
    ctx = tg.Context(0)
    off, tgt, tid = bench.build_inputs(cfg, 0)
    g = tg.CsrGraph(off, tgt)
    scores = tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tid, ctx=ctx)
    perm = tg.permutation_from_scores(scores, ctx=ctx)
    rg = tg.reorder_graph(g, perm, ctx=ctx)
    gt = tg.transpose(rg, ctx=ctx)
    del rg, g
    new_tid = np.sort(perm.new_id_of[tid.ids])
    sampler = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(new_tid, 7, 0)
    lists = sampler.batches(order, cfg["fanouts"], cfg["batch"], 7, 0, 0, args.batches)
    offs = np.zeros(len(lists) + 1, np.uint64)
    offs[1:] = np.cumsum([len(x) for x in lists])
    np.savez(cache_path(args.config), perm=perm.new_id_of, ids=np.concatenate(lists), offs=offs)
    torch.cuda.synchronize()
    print(f"prep: {len(lists)} minibatches cached in {cache_path(args.config)}")


def k8(args):
    import torch
    from paper_2111_05894_b200 import tiergraph as tg
    cfg = bench.CONFIGS[args.config]
    z = np.load(cache_path(args.config))
    perm = tg.NodePermutation(z["perm"])
    ids, offs = z["ids"], z["offs"]
    n = len(perm.new_id_of)
    stream = torch.cuda.Stream(device=0)  # one stream for torch and tiergraph
    torch.cuda.set_stream(stream)
    ctx = tg.Context(0, stream=stream)
    t0 = time.time()
    feat, R, _ = bench.pin_features(cfg, ctx)
    lay = tg.plan_layout(n, bench.hot_fraction(cfg, 1), 0.0, 1, cfg["dim"], cfg["elem"],
                         (int(np.ceil(cfg["hot_per_gpu"] * n)) + 1) * R if "hot_per_gpu" in cfg
                         else 0)
    if cfg.get("row_cache_gb"):
        store = tg.TieredFeatureStore(None, perm, lay, 0, ctx=ctx, cold_mode=cfg["cold_mode"],
                                      place=False)
        store.place_rows(feat, (np.arange(n, dtype=np.uint64) % np.uint64(len(feat)))
                         .astype(np.uint32))
    else:
        store = tg.TieredFeatureStore(feat, perm, lay, 0, ctx=ctx,
                                      cold_mode=cfg.get("cold_mode", "reordered"))
    dev = torch.device("cuda", 0)
    lists = [torch.as_tensor(ids[offs[b]:offs[b + 1]].astype(np.int64), device=dev)
             for b in range(len(offs) - 1)]
    out = torch.empty((max(len(x) for x in lists), R), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    print(f"k8: store ready in {time.time()-t0:.1f}s", file=sys.stderr)
    for k in range(args.launches):
        flush.zero_()
        store.gather_rows_async(lists[k % len(lists)], out, cnt, err)
    torch.cuda.synchronize()
    assert int(err.item()) == -1
    print(f"k8: {args.launches} launches, counters {cnt.tolist()}")


def k3(args):
    import torch
    from paper_2111_05894_b200 import tiergraph as tg
    cfg = bench.CONFIGS[args.config]
    ctx = tg.Context(0)
    off, tgt, tid = bench.build_inputs(cfg, 0)
    g = tg.CsrGraph(off, tgt)
    g.device(ctx)
    for _ in range(args.launches):
        tg.weighted_reverse_pagerank(g, tg.PagerankConfig(), tid, ctx=ctx)
    torch.cuda.synchronize()
    print("k3: done")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["prep", "k8", "k3"])
    ap.add_argument("--config", default="c3", choices=sorted(bench.CONFIGS))
    ap.add_argument("--batches", type=int, default=16)
    ap.add_argument("--launches", type=int, default=4)
    args = ap.parse_args()
    {"prep": prep, "k8": k8, "k3": k3}[args.what](args)


if __name__ == "__main__":
    main()
