"""Experiment: fixed cost of one synchronous tg_gather_rows call (1 row),
against an empty CUDA launch + stream synchronize, with the ids pinned or on
the device. Not part of the bench."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2111_05894_b200 import tiergraph as tg
    from paper_2111_05894_b200._lib import LIB
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = tg.Context(0, stream=s)
    n, dim = 100000, 100
    feat = np.zeros((n, dim), np.float32)
    perm = np.arange(n, dtype=np.uint64)
    lay = tg.plan_layout(n, 0.2, 0.0, 1, dim, 4)
    st = tg.TieredFeatureStore(feat, perm, lay, ctx=ctx)
    dev = torch.device("cuda", 0)
    out = torch.empty((16, dim * 4), dtype=torch.uint8, device=dev)
    pinned = tg.host_alloc(8).view(np.uint64)
    pinned[0] = 5
    rep = tg.TgReport() if hasattr(tg, "TgReport") else None
    from paper_2111_05894_b200._lib import TgReport
    r = TgReport()
    ids_d = torch.tensor([5], dtype=torch.int64, device=dev)

    def t_calls(fn, k=2000):
        for _ in range(100):
            fn()
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        return (time.perf_counter() - t0) / k * 1e6

    x = torch.zeros(1, device=dev)
    print(f"empty torch kernel + stream sync        : {t_calls(lambda: (x.add_(1), s.synchronize())):6.1f} us")
    print(f"tg_gather_rows, 1 id pinned, dst device : "
          f"{t_calls(lambda: LIB.tg_gather_rows(st.h, C.c_void_p(pinned.ctypes.data), 1, C.c_void_p(out.data_ptr()), C.byref(r))):6.1f} us")
    print(f"tg_gather_rows, 1 id device, dst device : "
          f"{t_calls(lambda: LIB.tg_gather_rows(st.h, C.c_void_p(ids_d.data_ptr()), 1, C.c_void_p(out.data_ptr()), C.byref(r))):6.1f} us")
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    print(f"tg_gather_rows_async 1 id + stream sync : "
          f"{t_calls(lambda: (st.gather_rows_async(ids_d, out, cnt, err), s.synchronize())):6.1f} us")
    a = C.c_void_p()
    print(f"cudaPointerGetAttributes x1 (via tg)    : n/a")


if __name__ == "__main__":
    main()
