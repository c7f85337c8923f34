"""Experiment: K8 at C3 scale (papers100M-shaped) — where do the ~177 us per
minibatch go? Times the gather for several hot fractions and load paths on
the same 40 minibatch id lists (L2 flushed per step). Not part of the bench."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import producers, tiergraph as tg
    cfg = dict(bench.CONFIGS["c3"])
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
    gt = producers.transpose(rg)
    del rg
    new_tid = np.sort(perm.new_id_of[tid.ids])
    sampler = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(new_tid, 7, 0)
    lists = [sampler.minibatch(order[b * 1024:(b + 1) * 1024], cfg["fanouts"], 7, 0, b)
             for b in range(40)]
    feat, R, _ = bench.pin_features(cfg)
    dev = torch.device("cuda", 0)
    ids_d = [torch.as_tensor(x.astype(np.int64), device=dev) for x in lists]
    maxu = max(len(x) for x in lists)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["bulk", "ldg"]
    colds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["reordered", "indirect"]
    for hot, cold in [(0.2, c) for c in colds]:
        lay = tg.plan_layout(n, hot, 0.0, 1, cfg["dim"], cfg["elem"])
        for mode in modes:
            st = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx, gather_mode=mode,
                                       cold_mode=cold)
            out = torch.empty((maxu, R), dtype=torch.uint8, device=dev)
            cnt = torch.zeros(3, dtype=torch.int64, device=dev)
            err = torch.full((1,), -1, dtype=torch.int64, device=dev)
            for k in range(3):
                st.gather_rows_async(ids_d[k], out, cnt, err)
            ts = []
            for k in range(len(lists)):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                st.gather_rows_async(ids_d[k], out, cnt, err)
                b.record()
                ts.append((a, b))
            torch.cuda.synchronize()
            ms = [a.elapsed_time(b) for a, b in ts]
            c = cnt.cpu().numpy()
            u = sum(len(x) for x in lists)
            print(f"hot={hot:.2f} cold={cold:9s} mode={mode:5s} avg {np.mean(ms)*1e3:8.1f} us min "
                  f"{np.min(ms)*1e3:8.1f} us  {u * R / (sum(ms) * 1e-3) / 1e9:7.1f} GB/s  "
                  f"host share {c[2] / max(c.sum(), 1):.4f}  per-step us "
                  f"{[round(x * 1e3) for x in ms[:12]]}", flush=True)
            st.close()


if __name__ == "__main__":
    main()
