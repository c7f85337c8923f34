"""Experiment: K1 (in-degree) timing on a config graph, host-timed per call.
Not part of the bench."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import tiergraph as tg
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    off, tgt, tid = bench.build_inputs(cfg, 0)
    g = tg.CsrGraph(off, tgt)
    g.device(ctx)
    out = torch.empty(len(off) - 1, dtype=torch.int64, device="cuda")
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tg.in_degrees(g, ctx=ctx, out=out)
        torch.cuda.synchronize()
        print(f"in_degrees {(time.perf_counter() - t0) * 1e6:.0f} us", flush=True)


if __name__ == "__main__":
    main()
