"""Experiment helper: the weighted reverse PageRank scores of a config graph,
saved as .npy (input for scripts/select_probe.py).
  python scripts/save_scores.py c3 /tmp/c3_scores.npy"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import bench
    from paper_2111_05894_b200 import tiergraph as tg
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    off, tgt, tid = bench.build_inputs(bench.CONFIGS[sys.argv[1]], 0)
    scores = tg.weighted_reverse_pagerank(tg.CsrGraph(off, tgt), tg.PagerankConfig(), tid, ctx=ctx)
    np.save(sys.argv[2], np.asarray(scores))
    print("saved", len(scores), "scores; range", float(np.min(scores)), float(np.max(scores)))


if __name__ == "__main__":
    main()
