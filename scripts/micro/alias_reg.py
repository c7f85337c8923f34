"""Probe: which cudaHostRegister of a memfd-aliased range fails (window 0, or a
second mapping of the same pages)? Not part of the bench."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_2111_05894_b200 import tiergraph as tg  # noqa: E402
from paper_2111_05894_b200._lib import LIB  # noqa: E402

libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
tg.default_context()
for gb in (1, 8):
    phys = gb << 30
    fd = os.memfd_create("probe", 0)
    os.ftruncate(fd, phys)
    base = libc.mmap(None, 3 * phys, 0, 0x02 | 0x20 | 0x4000, -1, 0)
    for k in range(3):
        r = libc.mmap(base + k * phys, phys, 3, 0x01 | 0x10, fd, 0)
        assert r == base + k * phys
    C.memset(base, 1, phys)
    for k in range(3):
        rc = LIB.tg_host_register(C.c_void_p(base + k * phys), phys)
        print(f"{gb} GB memfd window {k}: rc={rc} {LIB.tg_last_error().decode() if rc else ''}", flush=True)
    # control: private anonymous
    p = libc.mmap(None, phys, 3, 0x02 | 0x20, -1, 0)
    C.memset(p, 1, phys)
    rc = LIB.tg_host_register(C.c_void_p(p), phys)
    print(f"{gb} GB anonymous: rc={rc} {LIB.tg_last_error().decode() if rc else ''}", flush=True)
os.system("ulimit -l; grep -i -E 'memlock|Shmem' /proc/meminfo; cat /proc/sys/kernel/shmmax")
