"""Experiment: does a cold row cost fewer PCIe requests when only its whole
128 B lines are read from host memory? Times one minibatch's worth of random
zero-copy row reads (C2: 7,744 cold rows of a 1.96M-row region) for
400 B rows at a 512 B stride (today's padded cold tier), 384 B rows at a
512 B stride, and 384 B rows packed at a 384 B stride. Not part of the bench."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2111_05894_b200 import tiergraph as tg
    from paper_2111_05894_b200._lib import LIB
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    region = 1_960_000
    for rows in (7744, 30000):
        for stride, R in ((512, 400), (512, 384), (384, 384), (400, 400), (512, 512)):
            h = torch.empty(region * stride, dtype=torch.uint8, pin_memory=True)
            h.fill_(1)
            us = C.c_double()
            rc = LIB.tg_measure_host_rows_us(ctx.h, C.c_void_p(h.data_ptr()), region, stride, R,
                                             rows, 10, C.byref(us))
            assert rc == 0, LIB.tg_last_error()
            print(f"rows {rows:6d} stride {stride} R {R}: {us.value:7.1f} us "
                  f"{rows * R / us.value / 1e3:6.1f} GB/s  {rows / us.value:6.1f} rows/us", flush=True)
            del h


if __name__ == "__main__":
    main()
