"""Experiment: where K3's time goes on a config graph — a full step, the
longest row alone (its serial DADD chain), and the 8 longest rows alone.
Not part of the bench contract."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import tiergraph as tg
    from paper_2111_05894_b200._lib import LIB
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = tg.Context(0, stream=s)
    off, tgt, tid = bench.build_inputs(cfg, 0)
    n = len(off) - 1
    deg = np.diff(off.astype(np.int64))
    order = np.argsort(-deg, kind="stable")
    g = tg.CsrGraph(off, tgt)
    gh = g.device(ctx)
    dev = torch.device("cuda", 0)
    d = torch.empty(n, dtype=torch.int32, device=dev)
    na = torch.empty(n, dtype=torch.float64, device=dev)
    nb = torch.empty_like(na)
    sc = torch.empty_like(na)
    tid_d = torch.as_tensor(tid.ids.astype(np.int64), device=dev)
    assert LIB.tg_pagerank_prepare_async(ctx.h, gh, tid_d.data_ptr(), len(tid.ids), d.data_ptr(),
                                         na.data_ptr()) == 0

    def t_step(rb, re, reps=5):
        ts = []
        for _ in range(reps + 1):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            assert LIB.tg_pagerank_step_async(ctx.h, gh, d.data_ptr(), 0.85, na.data_ptr(),
                                              nb.data_ptr(), sc.data_ptr(), rb, re, 0) == 0
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return min(ts[1:])

    print(f"graph: {n} nodes, {len(tgt)} edges; longest rows {deg[order[:5]].tolist()}")
    if "full" in sys.argv:  # for ncu: a few full steps only
        print(f"full step: {t_step(0, n, 2):8.1f} us")
        return
    if "hubonly" in sys.argv:  # for an ncu capture of the longest row's CTA
        r = int(order[0])
        print(f"longest row alone: {t_step(r, r + 1, 2):8.1f} us")
        return
    print(f"full step                      : {t_step(0, n):8.1f} us")
    r = int(order[0])
    print(f"longest row alone ({deg[r]:6d} edges): {t_step(r, r + 1):8.1f} us "
          f"-> {t_step(r, r + 1) * 1e3 * 1.965 / deg[r]:.2f} cycles/edge at 1965 MHz")
    r2 = int(order[1])
    print(f"2nd row alone     ({deg[r2]:6d} edges): {t_step(r2, r2 + 1):8.1f} us")
    lo = n // 2
    print(f"rows [n/2, n) ({int(deg[lo:].sum())} edges): {t_step(lo, n):8.1f} us")
    print(f"rows [0, n/2) ({int(deg[:lo].sum())} edges): {t_step(0, lo):8.1f} us")
    # in-degree (K1) and the whole call
    ts = bench.time_events(torch, lambda: LIB.tg_in_degrees(ctx.h, gh, sc.data_ptr()), 5)
    print(f"tg_in_degrees (K1 + widen)     : {min(ts)*1e3:8.1f} us")


if __name__ == "__main__":
    main()
