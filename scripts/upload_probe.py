"""Experiment: tg_graph_create from pageable host u64 arrays (the first
PageRank call's upload), host-timed, with and without host-side narrowing
(TIERGRAPH_UPLOAD_NARROW). Not part of the bench.

  python scripts/upload_probe.py <n> <e> [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import subprocess
    n, e = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    if os.environ.get("_UP_CHILD") != "1":
        for mode in ("1", "0", "1"):
            env = dict(os.environ, _UP_CHILD="1", TIERGRAPH_UPLOAD_NARROW=mode)
            subprocess.run([sys.executable, __file__, str(n), str(e), str(reps)], env=env, check=True)
        return
    import torch
    from paper_2111_05894_b200 import tiergraph as tg
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    rng = np.random.default_rng(1)
    tgt = rng.integers(0, n, size=e, dtype=np.uint64)
    off = np.linspace(0, e, n + 1).astype(np.uint64)
    ts = []
    for _ in range(reps):
        g = tg.CsrGraph(off, tgt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.device(ctx)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        g.release()
    print(f"narrow={os.environ['TIERGRAPH_UPLOAD_NARROW']} n={n} e={e}: upload "
          + " ".join(f"{t * 1e3:.1f}" for t in ts) + " ms", flush=True)


if __name__ == "__main__":
    main()
