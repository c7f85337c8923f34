"""Experiment (not part of the bench contract): K3 step time on a config
graph under runtime knobs, each setting checked bit-identical to the first.

  python scripts/k3_probe.py c3 "TIERGRAPH_PR_PERSIST_MB=0" "TIERGRAPH_PR_PERSIST_MB=" ...
Each argument after the config is one setting: space-separated VAR=VALUE
pairs (an empty value unsets the variable); without arguments the settings
come from $K3_SETTINGS, ';'-separated."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import tiergraph as tg
    from paper_2111_05894_b200._lib import LIB
    cfg = bench.CONFIGS[sys.argv[1]]
    settings = sys.argv[2:] or os.environ.get("K3_SETTINGS", "").split(";")
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    off, tgt, tid = bench.build_inputs(cfg, 0)
    n, e = len(off) - 1, len(tgt)
    import numpy as np
    lens = np.diff(np.asarray(off, dtype=np.int64))
    for lo, hi in ((4096, None), (512, 4096), (0, 512)):
        m = (lens > lo) & ((lens <= hi) if hi else True)
        print(f"class len in ({lo}, {hi or 'inf'}]: {int(m.sum())} rows, {int(lens[m].sum())} edges",
              flush=True)
    indeg = np.bincount(np.asarray(tgt, dtype=np.int64), minlength=n)
    cum = np.cumsum(np.sort(indeg)[::-1])
    for k in (1 << 20, 1 << 22, 1 << 24, 1 << 25):
        print(f"top {k} in-degree nodes ({8 * k >> 20} MB of norm): {cum[min(k, n) - 1] / e:.3f} "
              f"of the gathers", flush=True)
    del indeg, cum, lens
    g = tg.CsrGraph(off, tgt)
    gh = g.device(ctx)
    fresh = os.environ.get("K3_FRESH_GRAPH") == "1"  # rebuild the device graph (and twin) per setting
    dev = torch.device("cuda", 0)
    tid_d = torch.as_tensor(tid.ids.astype("int64"), device=dev)
    ref = None
    iters = 5
    for st in settings:
        for kv in st.split():
            k, _, v = kv.partition("=")
            if v:
                os.environ[k] = v
            else:
                os.environ.pop(k, None)
        if fresh:
            g.release()
            torch.cuda.synchronize()
            gh = g.device(ctx)
        out = torch.empty(n, dtype=torch.float64, device=dev)
        ph = (C.c_double * (iters + 1))()
        steps = []
        clk = bench.ClockSampler(0)
        clk.__enter__()
        for _ in range(3):
            assert LIB.tg_weighted_reverse_pagerank_timed(ctx.h, gh, iters, 0.85, tid_d.data_ptr(),
                                                          len(tid.ids), out.data_ptr(), ph) == 0, \
                LIB.tg_last_error()
            steps.extend(ph[1:])
        clk.__exit__()
        mhz = sorted(c for _, c, _ in clk.samples)[len(clk.samples) // 2] if clk.samples else None
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out, ref))
        ms = statistics.mean(steps)
        per_step = [round(statistics.mean(steps[i::iters]), 3) for i in range(iters)]
        print(f"{st or '(default)':50s} step {ms:8.3f} ms  {e / ms / 1e6:7.1f} GTEPS/iter  "
              f"bit-identical {same}  sm {mhz} MHz  per step {per_step}", flush=True)


if __name__ == "__main__":
    main()
