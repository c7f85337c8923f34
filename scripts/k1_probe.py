"""Experiment: K1 (in-degree) timing on a config graph, host-timed per call,
one-pass atomic form vs binned form (TIERGRAPH_K1), results compared.
Not part of the bench.

  python scripts/k1_probe.py c3
"""
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
    e = len(tgt)
    outs = {}
    for mode in ("atomic", "binned"):
        if mode != "binned":
            os.environ["TIERGRAPH_K1"] = mode
        else:
            os.environ.pop("TIERGRAPH_K1", None)
        out = torch.empty(len(off) - 1, dtype=torch.int64, device="cuda")
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tg.in_degrees(g, ctx=ctx, out=out)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        outs[mode] = out
        best = min(ts[1:])
        print(f"K1 {mode:7s}: {best * 1e6:9.0f} us (median {sorted(ts[1:])[2] * 1e6:.0f}), "
              f"{4 * e / best / 1e12:.3f} TB/s of targets read", flush=True)
    print("equal:", all(bool(torch.equal(outs["atomic"], o)) for o in outs.values()), flush=True)


if __name__ == "__main__":
    main()
