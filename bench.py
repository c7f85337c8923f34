#!/usr/bin/env python
"""Benchmark of the data-tiering hot path on B200 (one JSON line on rank 0).

Metric (BASELINE.json): feature-gather GB/s & minibatches/s at 1/2/4/8 B200;
reverse-PageRank GTEPS. A "step" is one minibatch of the tiered gather (K8):
the reference's own sampled node-id list for that minibatch, gathered from
local HBM / peer HBM / pinned host memory into a contiguous HBM buffer.
`value` = gathered payload GB/s over all ranks (ids + features resident, L2
flushed between steps, per-step CUDA events on the launching stream, max over
ranks); `e2e` = the same through the synchronous C-ABI call with the ids in
pinned host memory (H2D inside the timed region) and the TrafficReport read
back (D2H). PageRank (5 iterations, in-degrees included) and the selection
sort are timed alongside and reported as sub-objects.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
Under torchrun (N>1) every rank gathers its own minibatch stream; the hot
tier is sharded across the ranks and read through CUDA-IPC peer pointers.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "feature-gather GB/s & minibatches/s at 1/2/4/8 B200; reverse-PageRank GTEPS"

CONFIGS = {
    "c1": dict(workload="C1: R-MAT 1M nodes / 16M draws, 128-d f32, 10% train, fanout (10,15), "
                        "batch 1024, hot 20%",
               nodes=1_000_000, draws=16_000_000, dim=128, elem=4, fanouts=[10, 15], batch=1024,
               train=0.10, hot=0.20),
    "c2": dict(workload="C2: ogbn-products-shaped R-MAT 2.45M nodes / 61.9M draws, 100-d f32, "
                        "10% train, fanout (15,10,5), batch 1024, hot 20%",
               nodes=2_450_000, draws=61_900_000, dim=100, elem=4, fanouts=[15, 10, 5], batch=1024,
               train=0.10, hot=0.20),
    # C3: BASELINE names no train fraction, fanout or batch for papers100M;
    # 10 %, (15,10,5) and 1024 are used and stated. The epoch is bounded to
    # max_batches minibatches; the cold rows get their own pinned copy in
    # new-id (score) order (45 GB): the most-read cold rows then share the
    # first GBs, which the GPU translates far more cheaply than random rows of
    # the 57 GB original (87.6 vs 102.6 us per minibatch, profiles/r01f).
    "c3": dict(workload="C3: ogbn-papers100M-shaped R-MAT 111M nodes / 1.6B draws, 128-d f32, "
                        "10% train, fanout (15,10,5), batch 1024, hot 20% sharded over the "
                        "ranks, cold rows via UVA from a pinned copy in new-id order",
               nodes=111_000_000, draws=1_600_000_000, dim=128, elem=4, fanouts=[15, 10, 5],
               batch=1024, train=0.10, hot=0.20, max_batches=512, cold_mode="reordered",
               cpu_gather=False),
    # C4: the hot tier is capped at 5% of the rows PER GPU (plan_layout's
    # per-device budget, tiering.cpp:87-96), sharded, so K = 5% x ranks. The
    # 374.8 GB fp16 matrix exceeds the box's 196 GB of host RAM (and the
    # driver maps at most ~RAM-size of host memory for the GPU, measured), so
    # the host side is a pinned row cache of P rows (`row_cache_gb`) holding
    # the reordered matrix wrapped every P rows, placed with
    # tg_store_place_rows: new id i reads cache row (i mod P). Graph,
    # PageRank, selection, sampling, layout and accounting run at full size;
    # parity checks the gathered bytes against that map.
    "c4": dict(workload="C4: MAG240M-shaped R-MAT 244M nodes / 1.7B draws, 768-d fp16, 10% train, "
                        "fanout (15,10,5), batch 1024, hot budget 5% of rows per GPU (sharded), "
                        "cold rows via UVA",
               nodes=244_000_000, draws=1_700_000_000, dim=768, elem=2, fanouts=[15, 10, 5],
               batch=1024, train=0.10, hot_per_gpu=0.05, max_batches=256, cold_mode="indirect",
               cpu_gather=False, row_cache_gb=80, fp16=True),
}


def config_dict(cfg, n, e, world):
    """The workload as both arms report it (identical dicts: the driver
    compares them). Arm-specific setup goes under the line's `setup` key."""
    return {"workload": cfg["workload"], "nodes": n, "edges_after_dedup": e,
            "row_bytes": cfg["dim"] * cfg["elem"], "dim": cfg["dim"],
            "elem_bytes": cfg["elem"], "hot_fraction": hot_fraction(cfg, world),
            "train_fraction": cfg["train"], "fanouts": list(cfg["fanouts"]),
            "batch": cfg["batch"], "epoch_minibatches_max": cfg.get("max_batches"),
            "rng": {"graph": 1, "train_ids": 3, "minibatches": 7, "epoch": 0},
            "l2": "inputs > L2: each step's rows are a fresh minibatch; the GPU arm also "
                  "flushes L2 (256 MB memset) between steps"}


def source_rows(cfg, inv):
    """new id -> row of the host feature fixture: the original matrix row
    inv[id] (reorder.cpp:113-115), or for C4 the row cache row (id mod P)."""
    if cfg.get("row_cache_gb"):
        n = len(inv)
        return np.arange(n, dtype=np.uint64) % np.uint64(cache_rows(cfg))
    return np.asarray(inv, np.uint64)


def hot_fraction(cfg, world):
    return cfg["hot"] if "hot" in cfg else min(1.0, cfg["hot_per_gpu"] * world)


def expected_rows(cfg, new_ids, inv):
    """Closed-form rows of the bench matrix for NEW ids: the original row
    inv[id]; for C4, row cache row (id mod P) (see CONFIGS["c4"])."""
    from paper_2111_05894_b200 import synth
    new_ids = np.asarray(new_ids, np.uint64)
    if cfg.get("row_cache_gb"):
        ids = new_ids % np.uint64(cache_rows(cfg))
    else:
        ids = inv[new_ids.astype(np.int64)]
    if cfg.get("fp16"):
        return synth.expected_rows_f16(ids, cfg["dim"])
    return synth.expected_rows(ids, cfg["dim"])


def cache_rows(cfg):
    R = cfg["dim"] * cfg["elem"]
    return int(cfg["row_cache_gb"] * (1 << 30) // R)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (the recipe's nvidia-smi clocks line, without the
    nvidia-smi start-up latency that would miss a sub-second region)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.stop = threading.Event()
        self.t = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons

            def run():
                while not self.stop.is_set():
                    try:
                        self.samples.append((time.perf_counter(),
                                             nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                             int(get_reasons(h))))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 2.0:
                time.sleep(0.001)
        except Exception as e:  # no NVML: report no samples
            log(f"clock sampler unavailable: {e}")
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self, t_begin=None, t_end=None):
        win = [x for x in self.samples
               if (t_begin is None or x[0] >= t_begin) and (t_end is None or x[0] <= t_end)]
        if len(win) < 3:
            win = self.samples
        reasons = set()
        for _, _, m in win:
            for bit, nm in self.REASONS.items():
                if m & bit:
                    reasons.add(nm)
        sm = [c for _, c, _ in win]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(win), "source": "NVML, 2 ms poll"}


# ----------------------------------------------------------------------------
def build_inputs(cfg, device, rank=0, world=1):
    """Synthetic graph (GPU R-MAT), train ids, features in pinned host memory."""
    from paper_2111_05894_b200 import producers, synth, tiergraph as tg
    t0 = time.time()
    off, tgt = synth.rmat_graph(cfg["nodes"], cfg["draws"], seed=1, device=f"cuda:{device}")
    n, e = len(off) - 1, len(tgt)
    tid = producers.draw_random_train_ids(n, int(n * cfg["train"]), 3)
    log(f"[rank {rank}] graph {n} nodes / {e} edges, {len(tid.ids)} train ids ({time.time()-t0:.1f}s)")
    return off, tgt, tid


def pin_features(cfg, ctx=None, dist=None, rank=0, tag=""):
    """The host feature fixture in pinned memory. Under torchrun (dist given)
    ONE copy per node: rank 0 fills a POSIX shared segment that every rank
    maps and registers, instead of one 57 GB copy per rank.
    Returns (rows array, R, segment or None)."""
    from paper_2111_05894_b200 import synth, tiergraph as tg
    n, dim = cfg["nodes"], cfg["dim"]
    R = dim * cfg["elem"]
    rows = cache_rows(cfg) if cfg.get("row_cache_gb") else n
    seg = None
    if dist is not None:
        name = f"/tg_feat_{tag}"
        if rank == 0:
            seg = tg.SharedHostSegment(name, rows * R, create=True)
        dist.barrier()
        if rank != 0:
            seg = tg.SharedHostSegment(name, rows * R, create=False)
        buf = seg.array
    else:
        buf = tg.host_alloc(rows * R)
    if dist is None or rank == 0:
        if cfg.get("row_cache_gb"):
            synth.test_features_f16_gpu(rows, dim, buf)
        elif n * R > (8 << 30):
            synth.test_features_pinned_gpu(n, dim, buf)
        else:
            synth.test_features(n, dim, out=buf)
    if dist is not None:
        dist.barrier()  # filled
    return buf.reshape(rows, R), R, seg


def time_events(torch, fn, reps, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return ts


def bench_pagerank(torch, tg, ctx, g, tid, n, e, iters=5, reps=5):
    """Whole weighted_reverse_pagerank call on device-resident data + the
    per-kernel prepare / SpMV-step device times for the roofline (CUDA events
    between the phases of the same call, tg_weighted_reverse_pagerank_timed).
    The one-time K3 relabelling (built with the device graph on first use,
    like the row schedule) is reported separately."""
    import ctypes as C
    from paper_2111_05894_b200._lib import LIB
    dev = torch.device("cuda", ctx.device)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    tid_d = torch.as_tensor(tid.ids.astype(np.int64), device=dev)
    cfgp = tg.PagerankConfig(iters, 0.85)
    gh = g.device(ctx)
    rl, rl_ms = C.c_int(), C.c_double()
    assert LIB.tg_pagerank_relabel_info(ctx.h, gh, C.byref(rl), C.byref(rl_ms)) == 0
    ts = time_events(torch, lambda: tg.weighted_reverse_pagerank(g, cfgp, tid_d, ctx=ctx, out=out),
                     reps)
    ms = min(ts)
    sc = torch.empty_like(out)
    ph = (C.c_double * (iters + 1))()
    step_ms, prep_ms = [], []
    for _ in range(reps):
        assert LIB.tg_weighted_reverse_pagerank_timed(ctx.h, gh, iters, 0.85, tid_d.data_ptr(),
                                                      len(tid.ids), sc.data_ptr(), ph) == 0
        prep_ms.append(ph[0])
        step_ms.extend(ph[1:])
    assert sc.cpu().numpy().tobytes() == out.cpu().numpy().tobytes()
    return out, ms, statistics.mean(step_ms), statistics.mean(prep_ms), \
        {"relabelled": bool(rl.value), "build_ms": round(rl_ms.value, 3)}


def bench_pagerank_e2e(torch, tg, ctx, off, tgt, tid, want_d):
    """weighted_reverse_pagerank through the public API with HOST buffers
    (u64 CSR + train ids in, f64 scores out), host-timed: the first call on a
    new CsrGraph uploads it (u32 narrowing, K1, the K3 schedule and relabel
    twin) and the later calls reuse the cached device copy, as the C++
    drop-in's device-graph cache does."""
    g = tg.CsrGraph(off, tgt)
    cfgp = tg.PagerankConfig(5, 0.85)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = tg.weighted_reverse_pagerank(g, cfgp, tid, ctx=ctx)
        ts.append(time.perf_counter() - t0)
    same = bool(s.tobytes() == want_d.cpu().numpy().tobytes())
    g.release()
    e = len(tgt)
    return {"first_call_s": round(ts[0], 4), "cached_call_s": round(min(ts[1:]), 4),
            "gteps_first_call": round(5 * e / ts[0] / 1e9, 3),
            "gteps_cached": round(5 * e / min(ts[1:]) / 1e9, 3),
            # the host arrays handed to the API (u64) ...
            "h2d_bytes_first_call": int(8 * (len(off) + len(tgt) + len(tid.ids))),
            # ... and what crosses PCIe: targets >= 4M narrowed to u32 by the
            # host cores on their way into the pinned pipeline (tg_graph_create)
            "pcie_h2d_bytes_first_call": int(8 * (len(off) + len(tid.ids)) + sum(
                min(32 << 20, e - b) * (4 if min(32 << 20, e - b) * 8 >= (32 << 20) else 8)
                for b in range(0, e, 32 << 20))),
            "d2h_bytes": int(8 * (len(off) - 1)), "bit_exact": same,
            "how": "tiergraph.weighted_reverse_pagerank(CsrGraph(host u64 arrays), host train "
                   "ids) -> host f64 scores, host perf_counter around each call"}


def bench_pagerank_multi(torch, tg, ctx, g, tid, single, dist, reps=3):
    """Row-partitioned PageRank over all ranks, device-timed, max over ranks,
    checked bit-exact against this rank's single-GPU run, with both
    exchanges: the baseline (an NCCL all-gather of the `norm` blocks after
    every step) and the fused one (each step's epilogue stores its rows into
    every rank's vector over CUDA-IPC peer memory; a device arrival barrier
    replaces the collective)."""
    from paper_2111_05894_b200 import distributed as D
    cfgp = tg.PagerankConfig(5, 0.85)
    ex = D.PeerExchangePagerank(g, ctx)
    runs = {"allgather": lambda: D.weighted_reverse_pagerank_multi(g, cfgp, tid, ctx=ctx),
            "fused_p2p": lambda: D.weighted_reverse_pagerank_ipc(g, cfgp, tid, ctx=ctx, exchange=ex)}
    res = {}
    for name, fn in runs.items():
        out = fn()  # warm (row schedule, IPC mappings)
        ts = []
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            out = fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        t = allreduce(dist, [min(ts)], single.device, dist.ReduceOp.MAX)
        same = allreduce(dist, [int(torch.equal(out, single))], single.device, dist.ReduceOp.MIN)
        res[name] = (float(t[0]), bool(same[0]))
    dist.barrier()
    ex.close()
    return res


def bench_structure(torch, tg, producers, ctx, gt, new_tid, cfg, lay, lists, nbat, rank, world,
                    dist, tag):
    """Graph-structure tiering: the
    sampler's transposed graph placed by the features' TierLayout (hot rows
    in HBM, sharded over the ranks and read over CUDA-IPC peer pointers;
    cold rows in ONE pinned host copy per node). Checked bit-exact against
    the whole-graph sampler's lists; reports the sampler rate and the
    neighbour-id bytes each tier served over this rank's share of the epoch
    against the untiered case (every id read over PCIe from host memory, as
    in the paper's CPU-resident graph)."""
    import ctypes as C
    from paper_2111_05894_b200._lib import LIB
    seg = None
    t0 = time.time()
    if world > 1:
        nb = producers.TieredGraph.cold_bytes(gt.offsets, lay)
        name = f"/tg_sgcold_{tag}"
        if rank == 0:
            seg = tg.SharedHostSegment(name, nb, create=True)
        dist.barrier()
        if rank != 0:
            seg = tg.SharedHostSegment(name, nb, create=False)
    sg = producers.TieredGraph(gt.offsets, gt.targets, lay, rank, ctx=ctx, cold=seg,
                               fill=(rank == 0))
    opened = []
    if world > 1:
        dist.barrier()  # rank 0 wrote the shared cold rows
        h = (C.c_uint8 * 64)()
        assert LIB.tg_ipc_get_handle(C.c_void_p(sg.local_base), h) == 0, LIB.tg_last_error()
        allh = [None] * world
        dist.all_gather_object(allh, bytes(h))
        for d in range(world):
            if d == rank:
                continue
            hb = (C.c_uint8 * 64).from_buffer_copy(allh[d])
            p = C.c_void_p()
            assert LIB.tg_ipc_open_handle(ctx.h, hb, C.byref(p)) == 0, LIB.tg_last_error()
            sg.set_peer(d, p.value)
            opened.append(p.value)
    build_s = time.time() - t0
    s = producers.GpuSampler(sg, ctx=ctx)
    order = producers.epoch_order(new_tid, 7, 0)
    B = cfg["batch"]
    per = max(1, nbat // world)  # a contiguous block of the epoch's batches per rank
    mine = list(range(rank * per, min(nbat, (rank + 1) * per)))
    chunk = min(len(mine), 32)
    s.batches(order, cfg["fanouts"], B, 7, 0, mine[0], chunk, device=True)  # warm
    s.structure_reads(reset=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t_s = time.perf_counter()
    ok = True
    for b0 in range(mine[0], mine[-1] + 1, chunk):  # members left in HBM, as the sampler leg
        s.batches(order, cfg["fanouts"], B, 7, 0, b0, min(chunk, mine[-1] + 1 - b0), device=True)
    torch.cuda.synchronize()
    el = time.perf_counter() - t_s
    reads = s.structure_reads(reset=True)
    for b in mine[:4]:  # spot check against the whole-graph sampler's lists
        ok &= bool(np.array_equal(s.batches(order, cfg["fanouts"], B, 7, 0, b, 1)[0], lists[b]))
    info = sg.info()
    vals = [float(reads[0]), float(reads[1]), float(reads[2]), el, float(ok)]
    if dist:
        vals = allreduce(dist, vals[:3], torch.device("cuda", ctx.device)) + \
            allreduce(dist, [el], torch.device("cuda", ctx.device), dist.ReduceOp.MAX) + \
            allreduce(dist, [float(ok)], torch.device("cuda", ctx.device), dist.ReduceOp.MIN)
    s.close()
    if dist:
        dist.barrier()
    for p in opened:
        LIB.tg_ipc_close_handle(C.c_void_p(p))
    sg.close()
    if dist:
        dist.barrier()
    if seg is not None:
        seg.close()
    r0, r1, r2, el, ok = vals
    tot = r0 + r1 + r2
    return {"minibatches_per_s": round(len(mine) * world / el, 1), "minibatches": len(mine) * world,
            "bit_exact_vs_whole_graph": bool(ok),
            "neighbour_id_bytes": {"local_hbm": int(4 * r0), "peer_hbm": int(4 * r1),
                                   "host_pcie": int(4 * r2), "untiered_host_pcie": int(4 * tot)},
            "pcie_reduction": round(1 - r2 / max(tot, 1), 4),
            "placement": dict(info, build_s=round(build_s, 2)),
            "how": "tg_sampler_create_tiered over tg_sgraph (csrc/structure.cu): row v of the "
                   "transposed reordered graph where resolve(v) puts feature row v; "
                   "tg_sample_batches over a contiguous block of the epoch's minibatches per "
                   "rank, 32 per call, members left in HBM, host-timed, max over ranks"}


def allreduce(dist, vals, device, op=None):
    """All-reduce a few host numbers (fp64) over the ranks; on the gloo
    plumbing of the shared-GPU test mode the tensor stays on the host."""
    import torch
    dev = device if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op if op is not None else dist.ReduceOp.SUM)
    return t.tolist()


def exchange_peers(torch, tg, store, rank, world):
    """CUDA-IPC handles of every rank's HBM region -> the combined-tensor table."""
    import ctypes as C
    import torch.distributed as dist
    from paper_2111_05894_b200._lib import LIB
    h = (C.c_uint8 * 64)()
    assert LIB.tg_ipc_get_handle(C.c_void_p(store.local_base), h) == 0, LIB.tg_last_error()
    mine = bytes(h)
    allh = [None] * world
    dist.all_gather_object(allh, mine)
    opened = []
    for d in range(world):
        if d == rank:
            continue
        hb = (C.c_uint8 * 64).from_buffer_copy(allh[d])
        p = C.c_void_p()
        assert LIB.tg_ipc_open_handle(store.ctx.h, hb, C.byref(p)) == 0, LIB.tg_last_error()
        store.set_peer(d, p.value)
        opened.append(p.value)
    return opened


def run_ours(args):
    import torch
    from paper_2111_05894_b200 import producers, tiergraph as tg

    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TG_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo plumbing (NCCL
    # refuses two ranks on one GPU) -- exercises the multi-process path
    # (CUDA-IPC peer tables, row-partitioned PageRank, max-over-ranks timing)
    # on a one-GPU box. Not a scaling measurement.
    share = world > 1 and os.environ.get("TG_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream(device=local)  # one non-default stream for torch and tiergraph
    torch.cuda.set_stream(stream)
    ctx = tg.Context(local, stream=stream)
    hbm_peak, hbm_src = measured_peaks()

    off, tgt, tid = build_inputs(cfg, local, rank, world)
    n, e = len(off) - 1, len(tgt)
    g = tg.CsrGraph(off, tgt)
    g.device(ctx)

    # ---- hot path A: PageRank + selection (device-resident graph)
    scores_d, pr_ms, step_ms, prep_ms, relabel = bench_pagerank(torch, tg, ctx, g, tid, n, e)
    indeg_out = torch.empty(n, dtype=torch.int64, device=torch.device("cuda", local))
    indeg_ms = min(time_events(torch, lambda: tg.in_degrees(g, ctx=ctx, out=indeg_out), 3))
    import ctypes as _C
    from paper_2111_05894_b200._lib import LIB as _LIB
    floor_us = _C.c_double()
    assert _LIB.tg_measure_gather_floor_us(ctx.h, g.device(ctx), 5, _C.byref(floor_us)) == 0
    floor_us = floor_us.value
    floor0_us = _C.c_double()  # the same in the graph's own labelling
    assert _LIB.tg_measure_gather_floor_us(ctx.h, g.device(ctx), -5, _C.byref(floor0_us)) == 0
    floor0_us = floor0_us.value
    pr_e2e = bench_pagerank_e2e(torch, tg, ctx, off, tgt, tid, scores_d)
    pr_multi = None
    if world > 1:
        pr_multi = bench_pagerank_multi(torch, tg, ctx, g, tid, scores_d, dist)
    dev = torch.device("cuda", local)
    perm_d = torch.empty(n, dtype=torch.int64, device=dev)
    sel = time_events(torch, lambda: tg.permutation_from_scores(scores_d, ctx=ctx, out=perm_d), 3)
    scores = scores_d.cpu().numpy()
    perm = tg.NodePermutation(perm_d.cpu().numpy().view(np.uint64))

    # ---- reordered graph -> the reference's minibatch schedule (host producer)
    t0 = time.time()
    rg = tg.reorder_graph(g, perm, ctx=ctx)
    # the PageRank device graph (and its relabelled twin) and the sort / staging
    # scratch are done with: free them before the largest allocations (C4:
    # the transpose stages 2 x 15 GB of u64 CSR and sorts 1.7G edges)
    g.release()
    ctx.trim()
    torch.cuda.empty_cache()
    gt = tg.transpose(rg, ctx=ctx)  # on the device (csr_graph.cpp:67-80)
    transpose_ok = None
    if world == 1 and not args.no_cpu_baseline and cfg.get("cpu_gather", True):
        import oracle  # checker only: the reference's transpose of the same graph
        chk = oracle.ref() or oracle.port()
        t_off, t_tgt = chk.transpose(rg.offsets, rg.targets)
        transpose_ok = bool(np.array_equal(t_off, gt.offsets) and np.array_equal(t_tgt, gt.targets))
    del rg
    new_tid = np.sort(perm.new_id_of[tid.ids])
    # the epoch's minibatch id lists, sampled on the GPU (csrc/sampling.cu,
    # bit-identical to the reference's build_minibatch); spot-checked against
    # the host restatement
    sampler = producers.GpuSampler(tg.CsrGraph(gt.offsets, gt.targets), ctx=ctx)
    order = producers.epoch_order(new_tid, 7, 0)
    B = cfg["batch"]
    nbat = (len(order) + B - 1) // B
    if cfg.get("max_batches"):
        nbat = min(nbat, cfg["max_batches"])
    sampler.batches(order, cfg["fanouts"], B, 7, 0, 0, 1)  # warm
    # the sampler's own rate: member lists left in HBM (what the gather reads)
    chunk = min(nbat, 32)
    sampler.batches(order, cfg["fanouts"], B, 7, 0, 0, chunk, device=True)
    torch.cuda.synchronize()
    reps_s = []
    for _ in range(3):  # the median of 3 passes over the epoch (host-timed)
        t_s = time.perf_counter()
        for b0 in range(0, nbat, chunk):
            sampler.batches(order, cfg["fanouts"], B, 7, 0, b0, min(chunk, nbat - b0), device=True)
        reps_s.append(time.perf_counter() - t_s)
    sample_dev_s = statistics.median(reps_s)
    # the whole epoch with every member list copied to host memory
    t_s = time.perf_counter()
    lists = sampler.batches(order, cfg["fanouts"], B, 7, 0, 0, nbat)
    sample_s = time.perf_counter() - t_s
    host_check = producers.epoch_minibatches(gt, new_tid, cfg["fanouts"], B, seed=7, epoch=0,
                                             max_batches=2)
    sampler_ok = all(np.array_equal(a, b) for a, b in zip(host_check, lists))
    mine = lists[rank::world]
    log(f"[rank {rank}] {len(lists)} minibatches/epoch sampled on the GPU "
        f"(avg {np.mean([len(l) for l in lists]):.0f} ids) in {time.time()-t0:.1f}s")

    # ---- tiered store: hot rows in HBM (sharded across ranks), cold rows pinned
    cold_seg = None
    tag = f"{os.environ.get('MASTER_PORT', '0')}_{os.getppid()}"
    feat, R, feat_seg = pin_features(cfg, ctx, dist if world > 1 else None, rank, tag)
    hot = hot_fraction(cfg, world)
    budget = 0
    if "hot_per_gpu" in cfg:  # plan_layout's per-device HBM budget (tiering.cpp:87-96)
        budget = (int(np.ceil(cfg["hot_per_gpu"] * n)) + 1) * R
    lay = tg.plan_layout(n, hot, 0.0, world, cfg["dim"], cfg["elem"], budget)
    if cfg.get("row_cache_gb"):
        # the cache holds the rows in new-id (score) order, wrapping every P
        # rows, as a reorder_features'd matrix would (reorder.cpp:97-117)
        store = tg.TieredFeatureStore(None, perm, lay, rank, ctx=ctx,
                                      cold_mode=cfg.get("cold_mode", "reordered"), place=False,
                                      gather_mode=args.gather_mode)
        store.place_rows(feat, (np.arange(n, dtype=np.uint64) % np.uint64(len(feat)))
                         .astype(np.uint32))
    elif world > 1:
        # one cold tier per node: rank 0 writes it into a shared segment, the
        # other ranks map the same memory
        store = tg.TieredFeatureStore(None, perm, lay, rank, ctx=ctx,
                                      cold_mode=cfg.get("cold_mode", "reordered"), place=False,
                                      gather_mode=args.gather_mode)
        cname = f"/tg_cold_{tag}"
        if rank == 0:
            cold_seg = tg.SharedHostSegment(cname, store.cold_tier_bytes, create=True)
        dist.barrier()
        if rank != 0:
            cold_seg = tg.SharedHostSegment(cname, store.cold_tier_bytes, create=False)
        store.attach_cold(cold_seg, fill=rank == 0)
        if rank == 0:
            store.place(feat, perm)
        dist.barrier()
        if rank != 0:
            store.place(feat, perm)
    else:
        store = tg.TieredFeatureStore(feat, perm, lay, rank, ctx=ctx,
                                      cold_mode=cfg.get("cold_mode", "reordered"),
                                      gather_mode=args.gather_mode)
    if world > 1:
        exchange_peers(torch, tg, store, rank, world)
        dist.barrier()

    # ---- graph-structure tiering: the sampler over the tiered transposed graph
    structure = bench_structure(torch, tg, producers, ctx, gt, new_tid, cfg, lay, lists, nbat,
                                rank, world, dist, tag)

    # ---- device-resident per-step inputs
    nsteps = args.steps + args.warmup
    ids_d = [torch.as_tensor(mine[k % len(mine)].astype(np.int64), device=dev) for k in range(nsteps)]
    maxu = max(len(x) for x in mine)
    out_d = torch.empty((maxu, R), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(k):
        store.gather_rows_async(ids_d[k], out_d, cnt, err)

    clk = ClockSampler(local).__enter__()  # samples warm-up + timed region
    for k in range(args.warmup):
        flush.zero_()
        step(k)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = tg.kernel_launches()
    cnt.zero_()
    evs = []
    if True:
        torch.cuda.synchronize()
        t_begin = time.perf_counter()
        for k in range(args.warmup, nsteps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            step(k)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        t_end = time.perf_counter()
        if dist:
            dist.barrier()
    clk.__exit__(None, None, None)
    launches = tg.kernel_launches() - launches0
    step_times = [a.elapsed_time(b) for a, b in evs]
    t_ms = sum(step_times)
    assert int(err.item()) == -1, "gather reported an out-of-range id"
    counters = cnt.cpu().numpy()
    u_rows = sum(len(mine[k % len(mine)]) for k in range(args.warmup, nsteps))
    assert int(counters.sum()) == u_rows
    if dist:
        t_ms = allreduce(dist, [t_ms], dev, dist.ReduceOp.MAX)[0]
        tot = allreduce(dist, [u_rows, int(counters[0]), int(counters[1]), int(counters[2])], dev)
        u_all, cl, cp, ch = (int(x) for x in tot)
    else:
        u_all, cl, cp, ch = u_rows, int(counters[0]), int(counters[1]), int(counters[2])
    gbps = u_all * R / (t_ms * 1e-3) / 1e9
    mbps = args.steps * world / (t_ms * 1e-3)

    # ---- e2e: synchronous C-ABI, ids in pinned host memory, report read back
    pinned_ids = [tg.host_alloc(len(mine[k % len(mine)]) * 8).view(np.uint64) for k in range(nsteps)]
    for k in range(nsteps):
        pinned_ids[k][:] = mine[k % len(mine)]
    rep = tg.TrafficReport()
    for k in range(args.warmup):
        store.gather_rows(pinned_ids[k], out=out_d[:len(pinned_ids[k])], report=rep)
    torch.cuda.synchronize()
    # timed inside the library around each synchronous tg_gather_rows call
    # (the C/C++ caller's view), L2 flushed before each call
    e2e_t = store.time_gather_rows(pinned_ids[args.warmup:nsteps], out_d, rep, flush_l2=True)
    # the same through the Python mirror (interpreter overhead included)
    e2e_py = 0.0
    for k in range(args.warmup, nsteps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        store.gather_rows(pinned_ids[k], out=out_d[:len(pinned_ids[k])], report=rep)
        e2e_py += time.perf_counter() - t0
    if dist:
        e2e_t, e2e_py = allreduce(dist, [e2e_t, e2e_py], dev, dist.ReduceOp.MAX)
    e2e_gbps = u_all * R / e2e_t / 1e9
    e2e_py_gbps = u_all * R / e2e_py / 1e9
    h2d = u_rows * 8 / args.steps

    # ---- CPU->GPU bytes per epoch: K8 counters over this rank's share of the epoch
    ep = tg.TrafficReport()
    counts = np.zeros(n, np.uint64)
    for ids in mine:
        store.gather_rows(ids, out=out_d[:len(ids)], report=ep)
        counts[ids.astype(np.int64)] += np.uint64(1)  # lists are sorted-unique
    sim = tg.simulate_trace(tg.make_access_counter(counts), lay)
    host_epoch, total_epoch = ep.host_bytes, ep.local_bytes + ep.peer_bytes + ep.host_bytes
    if dist:
        host_epoch, total_epoch = (int(x) for x in allreduce(dist, [host_epoch, total_epoch], dev))

    # ---- C5: cache-ratio sweep of CPU->GPU bytes per epoch (replicated vs
    # sharded hot tier, 1/2/4/8 devices) from the whole epoch's access counter
    # (all ranks' minibatches), replayed on the GPU by hot_fraction_sweep
    # (tiering.cpp:177-202); the identity ordering is the score ordering
    # because rows are already in new-id order.
    sweep = None
    if rank == 0:
        all_counts = np.zeros(n, np.uint64)
        for ids in lists:
            all_counts[ids.astype(np.int64)] += np.uint64(1)
        acc = tg.make_access_counter(all_counts)
        ident = np.arange(n, dtype=np.uint64)
        fr = [0.0, 0.05, 0.1, 0.2, 0.25, 0.5, 1.0]
        sweep = {"fractions": fr, "epoch_minibatches": len(lists), "row_bytes": R}
        sweep["note"] = ("per-GPU HBM budget = fraction x N x row_bytes; replicated keeps the "
                         "same hot set on every GPU, sharded spreads min(1, D x fraction) of "
                         "the rows over D GPUs at the same per-GPU budget")
        for D in (1, 2, 4, 8):
            for mode in ("replicated", "sharded"):
                eff = fr if mode == "replicated" else [min(1.0, D * f) for f in fr]
                rep = 1.0 if mode == "replicated" else 0.0
                rows = tg.hot_fraction_sweep(acc, ident, eff, rep, D, cfg["dim"], cfg["elem"],
                                             ctx=ctx)
                host = [r.report.host_bytes for r in rows]
                sweep[f"{mode}_D{D}"] = {
                    "hot_fraction": eff, "host_bytes": host,
                    "reduction_vs_untiered": [round(1 - h / max(host[0], 1), 4) for h in host],
                    "peer_bytes": [r.report.peer_bytes for r in rows]}

    # ---- roofline of the dominant kernel (K8) — mixed HBM / NVLink / PCIe
    pcie_dma = host_link_dma_gbps(torch, dev)
    pcie_zc = tg.measure_host_read_gbps(ctx, 1 << 30, R if R % 16 == 0 else 512, 3)
    pcie_peak = max(pcie_dma, pcie_zc)
    nvl_peak = 770.0  # measured peer copy per direction (B200_PROFILING.md)
    per_launch = u_rows / args.steps
    alg_bytes = per_launch * (2 * R + 8)  # payload read + output write + ids
    t_launch = statistics.mean(step_times) * 1e-3
    frac_l, frac_p, frac_h = cl / max(u_all, 1), cp / max(u_all, 1), ch / max(u_all, 1)
    # a split cold row crosses PCIe as its whole 128 B lines (Hc bytes) and
    # reads its remainder from HBM (TG_COLD_SPLIT_TAIL)
    Hc = store.cold_host_bytes
    hbm_bytes = per_launch * (frac_l * R + frac_h * (R - Hc) + R + 8)
    t_hbm = hbm_bytes / (hbm_peak * 1e9)
    t_nvl = per_launch * frac_p * R / (nvl_peak * 1e9)
    t_pcie = per_launch * frac_h * Hc / (pcie_peak * 1e9)
    t_star = max(t_hbm, t_nvl, t_pcie)
    bound = ["hbm", "nvlink", "pcie"][int(np.argmax([t_hbm, t_nvl, t_pcie]))]
    achieved = alg_bytes / t_launch / 1e9
    peak_eff = alg_bytes / t_star / 1e9
    # the same K8 over each timed minibatch's COLD ids only (ids >= mb), L2
    # flushed: the PCIe part by itself, on the real access pattern
    cold_rows = int(round(per_launch * frac_h))
    cold_floor = None
    if cold_rows:
        cnt2 = torch.zeros(3, dtype=torch.int64, device=dev)
        cts = []
        for k in range(args.warmup, nsteps):
            cl = ids_d[k][ids_d[k] >= lay.multi_boundary]
            if not len(cl):
                continue
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            store.gather_rows_async(cl, out_d, cnt2, err)
            b.record()
            cts.append((a, b))
        torch.cuda.synchronize()
        cold_floor = statistics.mean(a.elapsed_time(b) for a, b in cts) * 1e3
    # the platform's own ceiling for that cold part: the same number of random
    # rows of the same cold tier by a plain copy kernel (host-memory path:
    # translation of the mapped region + PCIe), and the mixed roofline with
    # it in place of the link peak
    platform = None
    if cold_rows and not cfg.get("cold_mode") == "indirect":
        plat_us = store.measure_cold_rows_us(cold_rows, 10)
        t_plat = max(t_hbm, t_nvl, plat_us * 1e-6)
        platform = {"cold_rows_copy_us": round(plat_us, 2), "t_star_us": round(t_plat * 1e6, 2),
                    "frac": round(t_plat / t_launch, 4),
                    "what": "t* with the host term = a plain one-warp-per-row copy of the same "
                            "number of random rows of the same pinned cold tier (L2 flushed; "
                            "tg_store_measure_cold_rows_us): what this box's host-memory path "
                            "delivers for random rows (scripts/micro/cold_probe.cu: the cost "
                            "follows distinct 4 KB pages, independent of host page size and "
                            "copy engine, i.e. off-GPU translation)"}
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("gather_dram_bytes_per_launch")
        except Exception:
            traffic = None

    result = None
    if rank == 0:
        clocks = clk.summary(t_begin, t_end)
        pr_bytes_iter = 4 * (n + 1) + 4 * e + 8 * e + 4 * n + 8 * n
        result = {
            "metric": METRIC, "value": round(gbps, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (R-MAT graph, closed-form features, reference sampler id lists)",
            "config": config_dict(cfg, n, e, world),
            "setup": {"layout": lay.as_tuple(), "gather_mode": args.gather_mode,
                      "cold_mode": cfg.get("cold_mode", "reordered"),
                      "timing": "per-step CUDA events on the launching stream, L2 flushed "
                                "(256 MB memset) before every step, max over ranks",
                      "parallelism": f"{world} GPU(s), hot tier sharded" + (
                          ", features and cold tier: one POSIX shared segment per node, mapped "
                          "by every rank" if world > 1 else "")
                                     + (" (TEST MODE: all ranks share cuda:0, gloo plumbing; "
                                        "not a scaling number)" if share else "")},
            "minibatches_per_s": round(mbps, 1),
            "avg_ids_per_minibatch": round(u_all / max(args.steps * world, 1), 1),
            "hit_split": {"local": round(frac_l, 4), "peer": round(frac_p, 4), "host": round(frac_h, 4)},
            "e2e": {"value": round(e2e_gbps, 2), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": 32,
                    "how": "tg_gather_rows (synchronous C-ABI) called K times, each call timed "
                           "in the library (tg_time_gather_rows, steady_clock): ids from pinned "
                           "host memory read in place, rows into HBM, TrafficReport read back",
                    "python_mirror_gbps": round(e2e_py_gbps, 2)},
            "gpu_launches": int(launches),
            "roofline": {"bound": bound, "achieved": round(achieved, 2),
                         "peak": round(peak_eff, 2), "unit": "GB/s",
                         "frac": round(t_star / t_launch, 4), "traffic": traffic,
                         "kernel": "gather_bulk_kernel (K8: TMA bulk copies, cold tier " + (
                             "read in place)" if cfg.get("cold_mode") == "indirect"
                             else "128 B-padded)" if Hc == R
                             else f"split: {Hc} B of whole lines per row over PCIe, the last "
                                  f"{R - Hc} B from HBM)"),
                         "cold_bytes_over_pcie_per_row": int(Hc),
                         "algorithmic_bytes_per_launch": int(alg_bytes),
                         "mixed": {"hbm_gbs": hbm_peak, "hbm_src": hbm_src,
                                   "pcie_gbs": round(pcie_peak, 2),
                                   "pcie_src": f"measured live: max(DMA H2D {pcie_dma:.1f}, "
                                               f"zero-copy row read {pcie_zc:.1f})",
                                   "nvlink_gbs": nvl_peak, "t_star_us": round(t_star * 1e6, 2),
                                   "t_launch_us": round(t_launch * 1e6, 2)},
                         "platform": platform,
                         "cold_floor": None if cold_floor is None else {
                             "us": round(cold_floor, 2), "rows": cold_rows,
                             "frac": round(cold_floor / (t_launch * 1e6), 4),
                             "what": "K8 over each timed minibatch's cold ids only (ids >= "
                                     "multi_boundary, L2 flushed): the PCIe part by itself on "
                                     "the real access pattern, GPU address translation "
                                     "included; frac = cold-only / full launch (1.0 = the HBM "
                                     "rows are fully hidden)"}},
            "pagerank": {"gteps": round(5 * e / (pr_ms * 1e-3) / 1e9, 3), "ms": round(pr_ms, 4),
                         "iterations": 5, "edges": e,
                         "note": "device-resident u32 CSR; in-degrees (K1) are built with the "
                                 "device graph and reported separately as indeg_us",
                         "indeg_us": round(indeg_ms * 1e3, 2),
                         "gteps_incl_indeg": round(5 * e / ((pr_ms + indeg_ms) * 1e-3) / 1e9, 3),
                         "multi_gpu": None if pr_multi is None else {
                             name: {"ranks": world, "ms": round(v[0], 4),
                                    "gteps": round(5 * e / (v[0] * 1e-3) / 1e9, 3),
                                    "bit_exact_vs_single_gpu": v[1],
                                    "exchange": {
                                        "allgather": "NCCL all_gather_into_tensor of norm row "
                                                     "blocks after every step",
                                        "fused_p2p": "K3 epilogue stores rows into every rank's "
                                                     "norm over CUDA-IPC peer memory + device "
                                                     "arrival barrier"}[name]}
                             for name, v in pr_multi.items()},
                         "relabel": dict(relabel, what=(
                             "K3 runs on a twin of the device graph whose rows are stored in "
                             "(class A by length, then length bucket, then in-degree) order and "
                             "whose nodes are labelled by storage row (sequential norm stores; "
                             "the most-gathered norms of each bucket share sectors); each row "
                             "keeps its own edge order, so sums are bit-identical; built once "
                             "per device graph like the row schedule (build_ms, not in `ms`)")),
                         "e2e": pr_e2e,
                         "spmv_step_us": round(step_ms * 1e3, 2),
                         "prepare_us": round(prep_ms * 1e3, 2),
                         "roofline": {"bound": "hbm", "kernel": "pr_step_kernel (K3)",
                                      "achieved": round(pr_bytes_iter / (step_ms * 1e-3) / 1e9, 1),
                                      "peak": hbm_peak, "unit": "GB/s",
                                      "frac": round(pr_bytes_iter / (step_ms * 1e-3) / 1e9 / hbm_peak, 4),
                                      "algorithmic_bytes_per_launch": pr_bytes_iter},
                         "gather_floor": {
                             "us": round(floor_us, 2),
                             "us_original_labels": round(floor0_us, 2),
                             "frac": round(floor_us / (step_ms * 1e3), 4),
                             "what": "the same E gathers norm[targets[e]] streamed over the same "
                                     "u32 CSR with no summation-order constraint "
                                     "(tg_measure_gather_floor_us): the memory-system floor of "
                                     "a K3 step on this graph; frac = floor / K3 step"}},
            "selection": {"ms": round(min(sel), 4), "keys": n},
            "sampling": {"minibatches_per_s": round(nbat / sample_dev_s, 1), "minibatches": nbat,
                         "how": "GPU build_minibatch (csrc/sampling.cu) over the epoch's batches, "
                                "32 per call back to back (tg_sample_batches: one host round trip "
                                "per call, 4 concurrent sampler lanes), member lists left in HBM; "
                                "host-timed, median of 3 passes over the epoch",
                         "with_host_copy_minibatches_per_s": round(nbat / sample_s, 1),
                         "matches_host_restatement": bool(sampler_ok),
                         "tiered_structure": structure},
            "epoch": {"minibatches": len(lists), "host_bytes_tiered": int(host_epoch),
                      "bytes_untiered": int(total_epoch),
                      "reduction": round(1 - host_epoch / max(total_epoch, 1), 4),
                      "equals_simulate_trace": bool(world > 1 or sim.host_bytes == ep.host_bytes)},
            "epoch_sweep": sweep,
            "clocks": clocks,
        }
        if cfg.get("row_cache_gb"):
            result["setup"]["host_row_cache"] = {
                "rows": cache_rows(cfg), "bytes": cache_rows(cfg) * R,
                "map": "new id i reads cache row (i mod rows), i.e. the reordered matrix "
                       "wrapped every `rows` rows: tg_store_place_rows",
                "why": "the 374.8 GB matrix exceeds the box's host RAM (196 GB)"}
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"], result["parity"] = cpu_baseline(
                cfg, off, tgt, tid, scores, perm, feat, R, lay, mine, store, out_d, torch,
                gt=gt, new_tid=new_tid, gpu_lists=lists)
            if transpose_ok is not None:
                result["parity"]["transpose_identical"] = transpose_ok
    if dist:
        dist.barrier()
        store.close()
        dist.barrier()  # every rank is done with the shared segments
        for seg in (cold_seg, feat_seg):
            if seg is not None:
                seg.close()
        dist.destroy_process_group()
    return result


def host_link_dma_gbps(torch, dev, nbytes=1 << 30):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        d.copy_(h, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


def cpu_baseline(cfg, off, tgt, tid, scores, perm, feat, R, lay, lists, store, out_d, torch,
                 gt=None, new_tid=None, gpu_lists=None):
    """The reference's CPU path (oracle/_ref, all host threads) on a bounded
    sample of the same workload, plus bit-exact parity of our results."""
    import oracle
    ref = oracle.ref()
    kind = "reference"
    if ref is None:
        ref, kind = oracle.port(), "port"
    cores = os.cpu_count() or 1
    parity = {}
    if kind == "reference":
        ref.set_worker_count(cores)
    # PageRank (whole run: seconds at C2, ~40 s at C3 on 16 cores)
    if kind == "reference":
        rg = ref.graph(off, tgt)  # the reference CsrGraph (construction not timed)
        t0 = time.perf_counter()
        want = rg.weighted_reverse_pagerank(tid.ids)
        pr_s = time.perf_counter() - t0
        del rg
    else:
        t0 = time.perf_counter()
        want = ref.weighted_reverse_pagerank(off, tgt, tid.ids)
        pr_s = time.perf_counter() - t0
    parity["pagerank_bit_exact"] = bool(want.tobytes() == scores.tobytes())
    parity["permutation_identical"] = bool(
        np.array_equal(ref.permutation_from_scores(want), perm.new_id_of))
    if kind != "reference":
        return ({"value": None, "unit": "GB/s", "cores": cores, "kind": kind,
                 "sample": "reference build missing"}, parity)
    ref.set_worker_count(cores)
    from paper_2111_05894_b200 import synth, tiergraph as tg
    moved, passes = 0, 0
    sample = lists[: max(1, min(len(lists), 24))]
    inv = np.empty(len(perm.new_id_of), np.uint64)
    inv[perm.new_id_of.astype(np.int64)] = np.arange(len(inv), dtype=np.uint64)
    if cfg.get("cpu_gather", True):
        # the reordered copy the reference would build (reorder_features)
        rf = oracle.RefFeatures(ref, feat.reshape(cfg["nodes"], R)).reordered(perm.new_id_of)
        how = "reference FeatureMatrix::row memcpy of reorder_features' copy"
    else:
        # no second 57 GB copy: the same rows read from the original matrix
        # through the inverse permutation (byte-identical, reorder.cpp:113-115)
        rf = oracle.RefFeaturesInv(ref, feat.reshape(-1, R), source_rows(cfg, inv))
        how = ("reference FeatureMatrix::row memcpy of the original matrix's row inv[id] "
               "(byte-identical to reorder_features' copy, which does not fit twice)")
    out = np.empty((max(len(x) for x in sample), R), np.uint8)
    rep = np.zeros(6, np.uint64)
    rf.gather(lay, sample[0], 0, out, rep)  # warm
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 3.0:  # a bounded ~3 s sample of CPU work
        for ids in sample:
            rf.gather(lay, ids, 0, out, rep)
            moved += len(ids) * R
        passes += 1
    cpu_s = time.perf_counter() - t0
    # gather parity on the last sampled minibatch: rows and report against
    # the reference, rows also against the closed-form fill
    ids = sample[-1]
    r = np.zeros(6, np.uint64)
    rf.gather(lay, ids, 0, out, r)
    mine = tg.TrafficReport()
    got = store.gather_rows(ids, report=mine)
    want = expected_rows(cfg, ids, inv)
    parity["gather_rows_bit_exact"] = bool(np.array_equal(got, out[: len(ids)]) and
                                           np.array_equal(got.view(want.dtype), want))
    if gt is not None:
        # the reference's own sampler on the host cores, and parity of the GPU sampler
        go_, gt_ = np.asarray(gt.offsets), np.asarray(gt.targets)
        t0 = time.perf_counter()
        ref_lists = ref.epoch_minibatches(go_, gt_, new_tid, cfg["fanouts"], cfg["batch"], 7, 0,
                                          max_batches=32)
        samp_s = time.perf_counter() - t0
        parity["gpu_sampler_bit_exact"] = bool(all(np.array_equal(a, b)
                                                   for a, b in zip(ref_lists, gpu_lists)))
    parity["traffic_report_equal"] = bool(np.array_equal(mine.as_array(), r))
    base = {"value": round(moved / cpu_s / 1e9, 3), "unit": "GB/s",
            "cores": cores, "kind": kind,
            "sample": (f"{passes} x {len(sample)} minibatches of the same epoch: {how} "
                       f"(reorder.cpp:113-115 pattern) + gather() accounting, {cores} OpenMP "
                       f"threads, {cpu_s:.2f}s"),
            "pagerank_gteps": round(5 * len(tgt) / pr_s / 1e9, 4),
            "minibatches_per_s": round(passes * len(sample) / cpu_s, 2),
            "sampling_minibatches_per_s": round(32 / samp_s, 2) if gt is not None else None,
            "pagerank_s": round(pr_s, 3)}
    return base, parity


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref: the unmodified reference sources, all host threads), rank 0
    only, on the same workload as the GPU arm. It never loads this repo's
    library: the fixtures (`synth`) are plain numpy/torch, and the package no
    longer loads libtiergraph_b200.so on import.

    Per run: the reference's PageRank (timed), permutation, reorder_graph and
    transpose produce the reorder_graph'd sampler input; the reference's
    build_minibatch lists give one step per minibatch. A step is the CPU byte
    gather of that minibatch (FeatureMatrix::row memcpy, reorder.cpp:113-115
    pattern, plus the reference gather() accounting). Where the reordered
    copy does not fit next to the original (C3, C4) the rows are read from the
    original fixture through the inverse permutation: byte-identical."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    ref = oracle.ref()
    cfg = CONFIGS[args.config]
    if ref is None:
        return {"impl": "reference", "unavailable": "oracle/_ref/libtgref.so was not built"}
    cores = os.cpu_count() or 1
    ref.set_worker_count(cores)
    from paper_2111_05894_b200 import synth
    t_all = time.time()
    dev = "cuda" if _cuda_available() else "cpu"
    off, tgt = synth.rmat_graph(cfg["nodes"], cfg["draws"], seed=1, device=dev)
    n, e = len(off) - 1, len(tgt)
    tid = ref.draw_random_train_ids(n, int(n * cfg["train"]), 3)
    log(f"[reference] graph {n} / {e} ({time.time()-t_all:.0f}s)")
    rg = ref.graph(off, tgt)  # the reference CsrGraph (construction not timed)
    t0 = time.perf_counter()
    scores = rg.weighted_reverse_pagerank(tid)
    pr_s = time.perf_counter() - t0
    del rg
    t0 = time.perf_counter()
    perm = ref.permutation_from_scores(scores)
    sel_s = time.perf_counter() - t0
    del scores
    ro, rt = ref.reorder_graph(off, tgt, perm)
    del off, tgt
    go, gt = ref.transpose(ro, rt)
    del ro, rt
    new_tid = np.sort(perm[tid])
    nsteps = args.steps + args.warmup
    nb_lists = min(nsteps, 64)
    t0 = time.perf_counter()
    lists = ref.epoch_minibatches(go, gt, new_tid, cfg["fanouts"], cfg["batch"], 7, 0,
                                  max_batches=nb_lists)
    samp_s = time.perf_counter() - t0
    del go, gt
    log(f"[reference] PageRank {pr_s:.1f}s, {len(lists)} minibatches in {samp_s:.1f}s "
        f"({time.time()-t_all:.0f}s)")
    R = cfg["dim"] * cfg["elem"]
    inv = np.empty(n, np.uint64)
    inv[perm.astype(np.int64)] = np.arange(n, dtype=np.uint64)
    if cfg.get("cpu_gather", True):
        feat = synth.test_features(n, cfg["dim"])
        rf = oracle.RefFeatures(ref, feat.view(np.uint8).reshape(n, R)).reordered(perm)
        del feat
        how = "FeatureMatrix::row memcpy of reorder_features' copy"
    else:
        if cfg.get("row_cache_gb"):
            P = cache_rows(cfg)
            feat = np.empty(P * R, np.uint8)
            synth.test_features_f16_gpu(P, cfg["dim"], feat, device=dev)
        else:
            feat = np.empty(n * R, np.uint8)
            synth.test_features_pinned_gpu(n, cfg["dim"], feat, device=dev)
        rf = oracle.RefFeaturesInv(ref, feat.reshape(-1, R), source_rows(cfg, inv))
        how = ("FeatureMatrix::row memcpy of the original matrix's row inv[id] (byte-identical "
               "to reorder_features' copy, which does not fit next to the original)")
    lay = ref.plan_layout(n, hot_fraction(cfg, 1), 0.0, 1, cfg["dim"], cfg["elem"],
                          (int(np.ceil(cfg["hot_per_gpu"] * n)) + 1) * R
                          if "hot_per_gpu" in cfg else 0)
    out = np.empty((max(len(x) for x in lists), R), np.uint8)
    rep = np.zeros(6, np.uint64)
    for k in range(args.warmup):
        rf.gather(lay, lists[k % len(lists)], 0, out, rep)
    t0 = time.perf_counter()
    moved = 0
    for k in range(args.warmup, nsteps):
        ids = lists[k % len(lists)]
        rf.gather(lay, ids, 0, out, rep)
        moved += len(ids) * R
    dt = time.perf_counter() - t0
    v = moved / dt / 1e9
    log(f"[reference] done ({time.time()-t_all:.0f}s)")
    return {"metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3 / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (R-MAT graph, closed-form features, reference sampler id lists)",
            "config": config_dict(cfg, n, e, world),
            "impl": "reference",
            "minibatches_per_s": round(args.steps / dt, 2),
            "avg_ids_per_minibatch": round(moved / R / max(args.steps, 1), 1),
            "pagerank": {"gteps": round(5 * e / pr_s / 1e9, 4), "s": round(pr_s, 3)},
            "selection": {"s": round(sel_s, 3), "keys": n},
            "sampling": {"minibatches_per_s": round(len(lists) / samp_s, 2),
                         "minibatches": len(lists)},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": cores,
                             "kind": "reference",
                             "sample": f"{args.steps} minibatches (the epoch's first, in order): "
                                       f"{how} + gather() accounting (reference build, "
                                       f"{cores} OpenMP threads)"},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather-mode", default="bulk+spread+dynamic",
                    help="K8 variant: ldg | bulk | l2pf, with +spread / +dynamic")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
