"""Experiment: per-segment timeline of K3's class-A kernel (TG_SEG_TRACE=1
prints it from the library) on a config graph. Not part of the bench."""
import os
import sys

import numpy as np

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
    tg.weighted_reverse_pagerank(g, tg.PagerankConfig(2, 0.85), tid, ctx=ctx)
    os.environ["TG_SEG_TRACE"] = "1"
    tg.weighted_reverse_pagerank(g, tg.PagerankConfig(2, 0.85), tid, ctx=ctx)


if __name__ == "__main__":
    main()
