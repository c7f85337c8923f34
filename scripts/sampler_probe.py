"""Experiment: the GPU sampler's per-kernel time on C2 (tg_sample_batches over
32 minibatches). Not part of the bench."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import producers, tiergraph as tg
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    off, tgt, tid = bench.build_inputs(cfg, 0)
    g = tg.CsrGraph(off, tgt)
    gt = tg.transpose(g, ctx=ctx)
    s = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(tid, 7, 0)
    s.batches(order, cfg["fanouts"], 1024, 7, 0, 0, 2)
    import ctypes as C
    from paper_2111_05894_b200._lib import LIB
    fo = np.asarray(cfg["fanouts"], np.uint32)
    od = torch.as_tensor(order.astype(np.int64), device="cuda")
    cap = 32 * 1_000_000
    md = torch.empty(cap, dtype=torch.int64, device="cuda")
    offs = np.empty(33, np.uint64)
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record(torch.cuda.Stream(device=0) if False else None)
        assert LIB.tg_sample_batches(s.h, od.data_ptr(), len(order), 1024, 0, 32, fo.ctypes.data,
                                     len(fo), 7, 0, md.data_ptr(), cap, offs.ctypes.data) == 0
        dt = time.perf_counter() - t0
        print(f"C-ABI only, device output: 32 minibatches {dt * 1e3:.2f} ms -> {32 / dt:.0f} mb/s",
              flush=True)
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lists = s.batches(order, cfg["fanouts"], 1024, 7, 0, 0, 32)
        dt = time.perf_counter() - t0
        print(f"32 minibatches: {dt * 1e3:.2f} ms -> {32 / dt:.0f} mb/s, "
              f"avg {np.mean([len(x) for x in lists]):.0f} ids", flush=True)


if __name__ == "__main__":
    main()
