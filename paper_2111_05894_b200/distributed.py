"""Multi-GPU reverse PageRank: row-partitioned K3 + all-gather of `norm`.

SURVEY §8(e): each rank owns one contiguous block of rows. Every Jacobi step
(reference `run_iterations`, scoring.cpp:50-74) computes `norm_out` (or, on
the last step, the scores) for the rank's rows only, then the blocks are
exchanged with one all-gather (NCCL over NVLink/NVSwitch on GPUs) so every
rank holds the full `norm` vector for the next step. A row's sum never
leaves its rank, so the result is bit-identical to the single-GPU run and to
the reference for any number of ranks (the reference's guarantee for any
worker count, parallel.hpp:5-7).

Two exchanges are provided:
  * `reverse_pagerank_partitioned` / `weighted_reverse_pagerank_multi`: one
    process per GPU, each holding only its edge-balanced row block; K1
    sharded (partial in-degrees + one all-reduce); an all-gather (NCCL) of the
    blocks after every step — the baseline;
  * `weighted_reverse_pagerank_peers`: the fused B200 path — each step's
    epilogue stores its rows straight into every rank's `norm` vector (P2P
    stores over NVLink/NVSwitch), and a device-side arrival barrier
    (tg_peer_barrier_async) replaces the collective, so the exchange overlaps
    the SpMV row by row. One process drives all ranks (one context each).

The all-gather driver is written against a small "stepper" interface so that the
partitioning and exchange logic runs unchanged over gloo in the CPU tests
(tests/test_distributed.py); the product stepper, `DeviceStepper`, launches
this library's kernels through the C-ABI (tg_pagerank_prepare_async /
tg_pagerank_step_async) and has no CPU path.
"""
from __future__ import annotations

import math
from typing import Optional, Tuple

import numpy as np


def edge_blocks(offsets, world: int) -> list:
    """Contiguous row blocks with near-equal EDGE counts: block r starts at the
    first row whose offset reaches ceil(r * E / world) (the same split as
    tg_row_blocks). Equal-row blocks put 3.4x the mean edge count on rank 0 of
    an R-MAT graph; these stay within a row's length of E/world."""
    off = np.asarray(offsets, np.uint64)
    n = max(len(off) - 1, 0)
    e = int(off[-1]) if n else 0
    b = [0]
    for r in range(1, world):
        if e == 0:
            b.append(n * r // world)
            continue
        want = (e * r + world - 1) // world
        b.append(min(max(int(np.searchsorted(off, np.uint64(want), side="left")), b[-1]), n))
    b.append(n)
    return [(b[r], b[r + 1]) for r in range(world)]


def row_blocks(n: int, world: int) -> Tuple[int, list]:
    """Equal row blocks (the fused IPC exchange's split): block r =
    [r*chunk, min(n, (r+1)*chunk))."""
    chunk = max(1, math.ceil(n / max(world, 1)))
    return chunk, [(min(n, r * chunk), min(n, (r + 1) * chunk)) for r in range(world)]


class DeviceStepper:
    """One rank's shard on its GPU, through the C-ABI: a ROW-BLOCK graph
    (tg_graph_create_rows: only this rank's rows and edges are uploaded), its
    partial in-degrees (the K1 shard), the K2 init from the summed in-degrees
    and the K3 steps over its rows."""

    def __init__(self, g, ctx, block):
        import ctypes as C
        import torch
        from . import tiergraph as tg
        from ._lib import LIB
        self.torch, self.tg, self.LIB = torch, tg, LIB
        self.ctx = ctx
        self.n = g.num_nodes()
        self.rb, self.re = block
        self.dev = torch.device("cuda", ctx.device)
        h = C.c_void_p()
        tg._check(LIB.tg_graph_create_rows(ctx.h, tg._ptr(g.offsets),
                                           tg._nonempty(g.targets, np.uint64), self.n,
                                           g.num_edges(), self.rb, self.re, C.byref(h)))
        self.gh = h

    def alloc(self, count: int):
        return self.torch.empty(count, dtype=self.torch.float64, device=self.dev)

    def partial_indeg(self):
        d = self.torch.empty(max(self.n, 1), dtype=self.torch.int32, device=self.dev)
        self.tg._check(self.LIB.tg_in_degrees_u32_async(self.ctx.h, self.gh, d.data_ptr()))
        self.sync()
        return d

    def init(self, tid_dev, ntid: int, indeg, norm0) -> None:
        self.indeg = indeg
        self.tg._check(self.LIB.tg_pagerank_init_async(
            self.ctx.h, self.n, tid_dev.data_ptr() if tid_dev is not None else None, ntid,
            indeg.data_ptr(), norm0.data_ptr()))

    def step(self, damp: float, nin, nout, sout, rb: int, re: int, last: bool) -> None:
        self.tg._check(self.LIB.tg_pagerank_step_async(
            self.ctx.h, self.gh, self.indeg.data_ptr(), float(damp), nin.data_ptr(),
            nout.data_ptr(), sout.data_ptr(), int(rb), int(re), int(last)))

    def sync(self) -> None:
        self.ctx.sync()

    def close(self) -> None:
        if self.gh:
            self.sync()
            self.LIB.tg_graph_destroy(self.gh)
            self.gh = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _exchange(out, stage, blocks, rank, group):
    """Every rank's block of `out` to every rank: one all-gather of blocks
    padded to the longest (NCCL over NVLink/NVSwitch on GPUs), then the blocks
    back in row order (one device copy each)."""
    import torch.distributed as dist
    chunk = len(stage) // len(blocks)
    rb, re = blocks[rank]
    mine = stage[rank * chunk:(rank + 1) * chunk]
    mine[:re - rb].copy_(out[rb:re])
    if out.is_cuda and dist.get_backend(group) != "nccl":
        # gloo plumbing (tests, shared-GPU bench mode): stage through the host
        h = stage.cpu()
        dist.all_gather_into_tensor(h, h[rank * chunk:(rank + 1) * chunk].clone(), group=group)
        stage.copy_(h)
    else:
        dist.all_gather_into_tensor(stage, mine.clone() if not stage.is_cuda else mine,
                                    group=group)
    for q, (b0, b1) in enumerate(blocks):
        if q != rank and b1 > b0:
            out[b0:b1].copy_(stage[q * chunk:q * chunk + (b1 - b0)])


def reverse_pagerank_partitioned(stepper, n: int, iterations: int, damp: float, tid=None,
                                 ntid: int = 0, group=None, blocks=None):
    """Runs the recurrence with rows split over the ranks of `group`
    (edge-balanced `blocks`, one per rank; the stepper holds this rank's) and
    returns the full score vector (length n) on every rank.

    K1 is sharded: every rank counts the in-degrees of its own edges and the
    counts are summed with one all-reduce. `tid` (a device tensor of train
    ids, or None for the unweighted recurrence) must be the same on every rank.
    """
    import torch
    import torch.distributed as dist
    if iterations < 1:
        from .tiergraph import DomainError
        raise DomainError("pagerank: iterations must be >= 1")  # scoring.cpp:43-44
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    rb, re = blocks[rank]
    indeg = stepper.partial_indeg()
    if world > 1:
        if indeg.is_cuda and dist.get_backend(group) != "nccl":
            h = indeg.cpu()
            dist.all_reduce(h, group=group)
            indeg.copy_(h)
        else:
            dist.all_reduce(indeg, group=group)  # K1 all-reduce (sum)
    a = stepper.alloc(max(n, 1))
    b = stepper.alloc(max(n, 1))
    scores = stepper.alloc(max(n, 1))
    chunk = max(1, max(b1 - b0 for b0, b1 in blocks))
    stage = stepper.alloc(chunk * world)
    stepper.init(tid, ntid, indeg, a)  # norm0 for every row (identical on every rank)
    x, y = a, b
    for it in range(iterations):
        last = it + 1 == iterations
        stepper.step(damp, x, y, scores, rb, re, last)
        out = scores if last else y
        if world > 1:
            stepper.sync()  # the step must land before the collective reads it
            _exchange(out, stage, blocks, rank, group)
        x, y = y, x
    stepper.sync()
    return scores[:n]


def weighted_reverse_pagerank_multi(g, cfg, tid, ctx=None, group=None):
    """scoring.hpp:45-46 on all ranks of `group` (one GPU per rank): each rank
    uploads only its edge-balanced row block."""
    import torch
    import torch.distributed as dist
    from . import tiergraph as tg
    ctx = ctx or tg.default_context()
    ids = tid.ids if isinstance(tid, tg.TrainIdSet) else tid
    if ids is None or len(ids) == 0:
        raise tg.DomainError("weighted reverse pagerank needs a non-empty train id set; "
                             "use reverse_pagerank when no nodes are labeled")  # scoring.cpp:89-91
    if not (0.0 < cfg.damp < 1.0):
        raise tg.DomainError(f"pagerank: damp must lie in (0,1), got {cfg.damp}")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    blocks = edge_blocks(g.offsets, world)
    st = DeviceStepper(g, ctx, blocks[rank])
    try:
        tid_d = torch.as_tensor(np.asarray(ids, np.uint64).astype(np.int64), device=st.dev)
        return reverse_pagerank_partitioned(st, g.num_nodes(), cfg.iterations, cfg.damp, tid_d,
                                            len(ids), group, blocks)
    finally:
        st.close()


def _push_blocks(LIB, tg, ctx_h, src_base: int, dst_bases, rb: int, re: int):
    """This rank's rows [rb, re) of a vector to every peer's copy of it: one
    contiguous copy per peer (copy engine over NVLink/NVSwitch)."""
    if re <= rb:
        return
    for d in dst_bases:
        tg._check(LIB.tg_memcpy_async(ctx_h, d + 8 * rb, src_base + 8 * rb, 8 * (re - rb)))


def weighted_reverse_pagerank_peers(g, cfg, tid, ctxs, timeout_check=True, exchange="copy"):
    """Partitioned PageRank with the FUSED exchange, one process driving
    several ranks (one context each; ranks may share a GPU): every step writes
    its rows straight into all ranks' `norm` vectors (P2P stores over NVLink
    between GPUs) and a device-side barrier replaces the all-gather
    (tg_pagerank_step_peers_async / tg_peer_barrier_async). Returns the full
    score vector of every rank (all identical, bit-exact to one GPU).
    `tid=None` runs the unweighted recurrence.

    exchange="copy" (default): the step writes its rows locally and the block
    is pushed to every peer as one contiguous copy before the barrier;
    "stores": the step's epilogue stores each row into every peer's vector
    (one 8 B remote store per row per peer)."""
    import ctypes as C
    import torch
    from . import tiergraph as tg
    from ._lib import LIB
    G = len(ctxs)
    n = g.num_nodes()
    if G >= 16:
        raise tg.DomainError("at most 15 peers")
    devs = [torch.device("cuda", c.device) for c in ctxs]
    for a in range(G):
        for b in range(G):
            if ctxs[a].device != ctxs[b].device:
                tg._check(LIB.tg_enable_peer_access(ctxs[a].device, ctxs[b].device))
    blocks = edge_blocks(g.offsets, G)
    gh = [g.device(c) for c in ctxs]
    deg = [torch.empty(max(n, 1), dtype=torch.int32, device=d) for d in devs]
    bufs = [[torch.empty(max(n, 1), dtype=torch.float64, device=d) for _ in range(3)] for d in devs]
    flags = [torch.zeros(2, dtype=torch.int32, device=d) for d in devs]  # [arrivals, err]
    ids = None if tid is None else (tid.ids if isinstance(tid, tg.TrainIdSet) else tid)
    for r, c in enumerate(ctxs):
        td = None if ids is None else torch.as_tensor(np.asarray(ids, np.uint64).astype(np.int64),
                                                      device=devs[r])
        tg._check(LIB.tg_pagerank_prepare_async(c.h, gh[r], None if td is None else td.data_ptr(),
                                                0 if ids is None else len(ids),
                                                deg[r].data_ptr(), bufs[r][0].data_ptr()))
        c.sync()  # keeps td alive until the prepare ran
    cur = 0
    for it in range(cfg.iterations):
        last = int(it + 1 == cfg.iterations)
        nxt = 1 - cur
        for r, c in enumerate(ctxs):
            peers = [q for q in range(G) if q != r]
            k = 2 if last else nxt
            rb, re = blocks[r]
            if exchange == "stores":
                pn = (C.c_void_p * 16)(*[bufs[q][nxt].data_ptr() for q in peers])
                ps = (C.c_void_p * 16)(*[bufs[q][2].data_ptr() for q in peers])
                tg._check(LIB.tg_pagerank_step_peers_async(
                    c.h, gh[r], deg[r].data_ptr(), float(cfg.damp), bufs[r][cur].data_ptr(),
                    bufs[r][nxt].data_ptr(), bufs[r][2].data_ptr(), rb, re, last, pn, ps,
                    len(peers)))
            else:
                tg._check(LIB.tg_pagerank_step_async(
                    c.h, gh[r], deg[r].data_ptr(), float(cfg.damp), bufs[r][cur].data_ptr(),
                    bufs[r][nxt].data_ptr(), bufs[r][2].data_ptr(), rb, re, last))
                _push_blocks(LIB, tg, c.h, bufs[r][k].data_ptr(),
                             [bufs[q][k].data_ptr() for q in peers], rb, re)
        for r, c in enumerate(ctxs):
            pf = (C.c_void_p * 16)(*[flags[q].data_ptr() for q in range(G) if q != r])
            tg._check(LIB.tg_peer_barrier_async(c.h, flags[r].data_ptr(), pf, G - 1,
                                                (it + 1) * (G - 1), flags[r].data_ptr() + 4))
        cur = nxt
    for c in ctxs:
        c.sync()
    if timeout_check and any(int(f[1].item()) for f in flags):
        raise tg.TierGraphError("peer barrier timed out")
    return [b[2][:n] for b in bufs]


class _DevView:
    """A device vector owned by this library, seen by torch (no copy)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "stream": None}


class PeerExchangePagerank:
    """The fused exchange with ONE PROCESS PER GPU (the form `bench.py` runs
    under torchrun): partitioned weighted reverse PageRank where every step's
    epilogue stores this rank's rows straight into all other ranks' `norm`
    (or score) vectors over NVLink/NVSwitch and a device-side arrival barrier
    replaces the all-gather -- `weighted_reverse_pagerank_peers` across
    processes.

    Each rank owns one library allocation (tg_device_alloc)
        [norm A | norm B | scores]  (n f64 each)  [arrivals u32, err u32]
    whose CUDA-IPC handle is exchanged once through the process group
    (all_gather_object, which also orders the zeroed counters before any
    arrival). Arrival counters only grow: the barrier target of a step is the
    running total of arrivals so far, so the object can run the recurrence any
    number of times without resetting them. Row sums never leave their rank,
    so the result is bit-identical to one GPU (scoring.cpp:50-74; any worker
    count, parallel.hpp:5-7).

    Safe reuse of the shared vectors (Jacobi ping-pong, scoring.cpp:71): a
    rank writes a peer's buffer X in step s only after the barrier of step
    s-1, and every rank finished its last read of X (step s-1 or earlier)
    before arriving there.
    """

    def __init__(self, g, ctx, group=None, exchange="copy"):
        import ctypes as C
        import torch
        import torch.distributed as dist
        from . import tiergraph as tg
        from ._lib import LIB
        self.tg, self.LIB, self.C, self.torch = tg, LIB, C, torch
        self.ctx, self.g = ctx, g
        self.gh = g.device(ctx)
        self.n = n = g.num_nodes()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world >= TG_MAX_PEERS + 1:
            raise tg.DomainError(f"at most {TG_MAX_PEERS} peers")
        self.exchange = exchange
        self.rb, self.re = edge_blocks(g.offsets, self.world)[self.rank]
        self.vec = ((max(n, 1) * 8 + 255) // 256) * 256
        nbytes = 3 * self.vec + 256
        base = C.c_void_p()
        tg._check(LIB.tg_device_alloc(ctx.h, nbytes, C.byref(base)))
        self.base = base.value
        self.dev = torch.device("cuda", ctx.device)
        self.deg = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        h = (C.c_uint8 * 64)()
        tg._check(LIB.tg_ipc_get_handle(C.c_void_p(self.base), h))
        handles = [bytes(h)] * self.world
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h), group=group)
        self.bases, self.opened = [], []
        for q in range(self.world):
            if q == self.rank:
                self.bases.append(self.base)
                continue
            hb = (C.c_uint8 * 64).from_buffer_copy(handles[q])
            p = C.c_void_p()
            tg._check(LIB.tg_ipc_open_handle(ctx.h, hb, C.byref(p)))
            self.bases.append(p.value)
            self.opened.append(p.value)
        self.arrivals = 0
        self.peers = [q for q in range(self.world) if q != self.rank]

    def _vec(self, base: int, k: int) -> int:
        return base + k * self.vec

    def _flag(self, base: int, k: int = 0) -> int:
        return base + 3 * self.vec + 4 * k

    def run(self, iterations: int, damp: float, tid_dev=None, ntid: int = 0):
        """Runs the recurrence (stream-ordered on the context, no host sync);
        returns the full score vector as a torch view of this rank's buffer,
        valid once the context stream has drained and until the next run."""
        C, LIB, tg = self.C, self.LIB, self.tg
        if iterations < 1:
            raise tg.DomainError("pagerank: iterations must be >= 1")  # scoring.cpp:43-44
        if not (0.0 < damp < 1.0):
            raise tg.DomainError(f"pagerank: damp must lie in (0,1), got {damp}")
        tg._check(LIB.tg_pagerank_prepare_async(
            self.ctx.h, self.gh, None if tid_dev is None else tid_dev.data_ptr(), ntid,
            self.deg.data_ptr(), self._vec(self.base, 0)))
        G = self.world
        pf = (C.c_void_p * 16)(*[self._flag(self.bases[q]) for q in self.peers])
        if G > 1:
            # entry barrier: no peer stores into this run's vectors before
            # every rank has finished reading the previous run's scores
            self.arrivals += G - 1
            tg._check(LIB.tg_peer_barrier_async(self.ctx.h, self._flag(self.base), pf, G - 1,
                                                self.arrivals, self._flag(self.base, 1)))
        cur = 0
        for it in range(iterations):
            last = int(it + 1 == iterations)
            nxt = 1 - cur
            if self.exchange == "stores":
                pn = (C.c_void_p * 16)(*[self._vec(self.bases[q], nxt) for q in self.peers])
                ps = (C.c_void_p * 16)(*[self._vec(self.bases[q], 2) for q in self.peers])
                tg._check(LIB.tg_pagerank_step_peers_async(
                    self.ctx.h, self.gh, self.deg.data_ptr(), float(damp),
                    self._vec(self.base, cur), self._vec(self.base, nxt),
                    self._vec(self.base, 2), self.rb, self.re, last, pn, ps, len(self.peers)))
            else:
                tg._check(LIB.tg_pagerank_step_async(
                    self.ctx.h, self.gh, self.deg.data_ptr(), float(damp),
                    self._vec(self.base, cur), self._vec(self.base, nxt),
                    self._vec(self.base, 2), self.rb, self.re, last))
                k = 2 if last else nxt
                _push_blocks(LIB, tg, self.ctx.h, self._vec(self.base, k),
                             [self._vec(self.bases[q], k) for q in self.peers], self.rb, self.re)
            if G > 1:
                self.arrivals += G - 1
                tg._check(LIB.tg_peer_barrier_async(
                    self.ctx.h, self._flag(self.base), pf, G - 1, self.arrivals,
                    self._flag(self.base, 1)))
            cur = nxt
        return self.torch.as_tensor(_DevView(self._vec(self.base, 2), self.n, "<f8"),
                                    device=self.dev)

    def timed_out(self) -> bool:
        """True when a device barrier gave up waiting (a peer never arrived)."""
        e = self.torch.as_tensor(_DevView(self._flag(self.base, 1), 1, "<u4"), device=self.dev)
        self.ctx.sync()
        return bool(int(e.cpu().item()))

    def close(self) -> None:
        self.ctx.sync()
        for p in self.opened:
            self.LIB.tg_ipc_close_handle(self.C.c_void_p(p))
        self.opened = []
        if self.base:
            self.LIB.tg_device_free(self.ctx.h, self.C.c_void_p(self.base))
            self.base = 0


TG_MAX_PEERS = 15


def weighted_reverse_pagerank_ipc(g, cfg, tid, ctx=None, group=None, exchange=None):
    """scoring.hpp:45-46 over all ranks of `group`, one process per GPU, with
    the fused P2P exchange. Pass a PeerExchangePagerank as `exchange` to reuse
    its buffers and IPC mappings across calls. Returns a copy of the scores."""
    import torch
    from . import tiergraph as tg
    ctx = ctx or tg.default_context()
    ids = tid.ids if isinstance(tid, tg.TrainIdSet) else tid
    if ids is None or len(ids) == 0:
        raise tg.DomainError("weighted reverse pagerank needs a non-empty train id set; "
                             "use reverse_pagerank when no nodes are labeled")  # scoring.cpp:89-91
    own = exchange is None
    ex = exchange or PeerExchangePagerank(g, ctx, group)
    tid_d = torch.as_tensor(np.asarray(ids, np.uint64).astype(np.int64), device=ex.dev)
    s = ex.run(cfg.iterations, cfg.damp, tid_d, len(ids))
    ex.ctx.sync()  # the last barrier has passed: every peer's rows have landed
    out = s.clone()
    torch.cuda.current_stream(ex.dev).synchronize()
    if ex.timed_out():
        raise tg.TierGraphError("peer barrier timed out")
    if own:
        ex.close()
    return out
