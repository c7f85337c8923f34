"""Experiment: where does the synchronous C-ABI gather (the bench's e2e) spend
the time K8 itself does not? C2 minibatches through tg_gather_rows with the
ids (a) in pinned mapped host memory, read in place by K8; (b) in pageable
host memory, staged to the device by a copy first; and (c) already on the
device (K8 alone, CUDA events). Not part of the bench."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import producers, tiergraph as tg
    cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
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
    gt = tg.transpose(rg, ctx=ctx)
    del rg, g
    new_tid = np.sort(perm.new_id_of[tid.ids])
    sampler = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(new_tid, 7, 0)
    lists = sampler.batches(order, cfg["fanouts"], cfg["batch"], 7, 0, 0, 60)
    feat, R, _ = bench.pin_features(cfg)
    lay = tg.plan_layout(n, 0.2, 0.0, 1, cfg["dim"], cfg["elem"])
    st = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx)
    dev = torch.device("cuda", 0)
    maxu = max(len(x) for x in lists)
    out = torch.empty((maxu, R), dtype=torch.uint8, device=dev)
    u = sum(len(x) for x in lists[5:])
    pinned = [tg.host_alloc(len(x) * 8).view(np.uint64) for x in lists]
    for p, x in zip(pinned, lists):
        p[:] = x
    pageable = [np.array(x, dtype=np.uint64) for x in lists]
    for name, ids in (("pinned, read in place", pinned), ("pageable, staged", pageable),
                      ("pinned, read in place", pinned)):
        st.time_gather_rows(ids[:5], out)
        t = st.time_gather_rows(ids[5:], out)
        print(f"tg_gather_rows, ids {name:22s}: {t / len(ids[5:]) * 1e6:7.1f} us per call "
              f"{u * R / t / 1e9:7.1f} GB/s", flush=True)
    ids_d = [torch.as_tensor(x.astype(np.int64), device=dev) for x in lists]
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
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
    ms = np.array([a.elapsed_time(b) for a, b in ts[5:]])
    print(f"K8 alone, device ids                 : {ms.mean() * 1e3:7.1f} us per launch "
          f"{u * R / (ms.sum() * 1e-3) / 1e9:7.1f} GB/s", flush=True)
    # launch + sync overhead: an empty list
    e = [np.zeros(1, np.uint64)] * 50
    t = st.time_gather_rows(e, out)
    print(f"tg_gather_rows of one id             : {t / 50 * 1e6:7.1f} us per call", flush=True)


if __name__ == "__main__":
    main()
