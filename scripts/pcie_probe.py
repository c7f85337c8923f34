"""Experiment: UVA zero-copy read GB/s of pinned mapped host memory by row size
(random row order, one warp per row, 16 B vectors) next to the DMA H2D copy
rate — the PCIe denominators of the K8 roofline. Not part of the bench contract."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2111_05894_b200 import tiergraph as tg
    torch.cuda.set_device(0)
    ctx = tg.Context(0)
    dev = torch.device("cuda", 0)
    print(f"DMA H2D 1 GiB: {bench.host_link_dma_gbps(torch, dev):.1f} GB/s")
    for R in (64, 128, 256, 400, 512, 768, 1024, 1536, 4096):
        v = tg.measure_host_read_gbps(ctx, 1 << 30, R, 5)
        print(f"zero-copy rows of {R:5d} B: {v:6.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
