"""Experiment (not part of the bench contract): hot-set selection (K4-K6,
tg_permutation_from_scores) on device-resident log-normal scores of n nodes,
host-timed around a synchronous call (the call syncs once for its error word),
plus a check that the result is a sort by (score desc, id asc).

  python scripts/select_probe.py [n=111000000 | scores.npy] [reps=5]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2111_05894_b200 import tiergraph as tg
    from paper_2111_05894_b200._lib import LIB
    src = sys.argv[1] if len(sys.argv) > 1 else "111000000"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    if src.endswith(".npy"):  # real scores (e.g. a config's PageRank output)
        import numpy as np
        s = torch.as_tensor(np.load(src), device=dev)
        n = s.numel()
    else:
        n = int(src)
        g = torch.Generator(device=dev).manual_seed(5)
        s = 1e-8 * torch.exp(2.5 * torch.randn(n, dtype=torch.float64, device=dev, generator=g))
        s[: n // 10] = s[n // 10: 2 * (n // 10)]  # exact duplicates: the id tie-break matters
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        assert LIB.tg_permutation_from_scores(ctx.h, s.data_ptr(), n, perm.data_ptr(),
                                              order.data_ptr()) == 0, LIB.tg_last_error()
        torch.cuda.synchronize()
        if r:
            ts.append(time.perf_counter() - t0)
    so = s[order]
    ok = bool((so[:-1] >= so[1:]).all())
    eq = so[:-1] == so[1:]
    ok &= bool((order[:-1][eq] < order[1:][eq]).all())
    ok &= bool((perm[order] == torch.arange(n, device=dev)).all())
    print(f"selection n={n}: {min(ts) * 1e3:.3f} ms (median {sorted(ts)[len(ts) // 2] * 1e3:.3f}), "
          f"sorted+tie-break+inverse {ok}", flush=True)


if __name__ == "__main__":
    main()
