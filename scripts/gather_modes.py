"""Experiment: K8 variants on the C2 workload (cold-tier load path x layout).

Times each gather mode on the same minibatch id lists (per-step CUDA events,
L2 flushed between steps) and checks every mode's output against the LDG
baseline byte for byte. Not part of the bench contract.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import producers, tiergraph as tg

    cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
    steps = 60
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
    gt = producers.transpose(rg)
    new_tid = np.sort(perm.new_id_of[tid.ids])
    lists = producers.epoch_minibatches(gt, new_tid, cfg["fanouts"], cfg["batch"], 7, 0,
                                        max_batches=steps)
    feat, R, _ = bench.pin_features(cfg)
    dev = torch.device("cuda", 0)
    ids_d = [torch.as_tensor(x.astype(np.int64), device=dev) for x in lists]
    maxu = max(len(x) for x in lists)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ref_out = None
    for hot in (cfg["hot"], 0.0, 1.0):
        lay = tg.plan_layout(n, hot, 0.0, 1, cfg["dim"], cfg["elem"])
        for mode in ("ldg", "ldg+spread", "bulk", "bulk+spread"):
            for pad in (False, True):
                st = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx, gather_mode=mode, pad128=pad)
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
                u = sum(len(x) for x in lists)
                k = len(lists) - 1
                check = out[:len(lists[k])].cpu().numpy()
                if ref_out is None or mode == "ldg" and not pad:
                    ref_out = check
                ok = np.array_equal(check, ref_out)
                print(f"hot={hot:.2f} mode={mode:11s} pad128={pad!s:5s} "
                      f"avg {np.mean(ms)*1e3:8.1f} us  min {np.min(ms)*1e3:8.1f} us  "
                      f"{u * R / (sum(ms) * 1e-3) / 1e9:8.1f} GB/s  match={ok}", flush=True)
                st.close()


if __name__ == "__main__":
    main()
