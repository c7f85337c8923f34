"""The multi-GPU decomposition, exercised over gloo on CPU (world_size 2 and 3).

paper_2111_05894_b200/distributed.py partitions the rows, runs one step per
rank and exchanges `norm` blocks with all_gather_into_tensor. Here the same
driver runs with a CPU stepper that restates the reference arithmetic
(scoring.cpp:59-70: IEEE division, left-to-right row sums, separately rounded
update — test infrastructure only), and the gathered scores must be
bit-identical to the reference build / C restatement for every rank count.
The GPU stepper is covered by tests/test_gpu_pagerank.py
(row-partitioned steps) and by the single-GPU multi-rank run below.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2111_05894_b200 import distributed as D


class CpuStepper:
    """One rank's shard: rows [rb, re) only (like tg_graph_create_rows)."""

    def __init__(self, off, tgt, block):
        self.off = off.astype(np.int64)
        self.tgt = tgt.astype(np.int64)
        self.n = len(off) - 1
        self.rb, self.re = block

    def alloc(self, count):
        return torch.zeros(count, dtype=torch.float64)

    def partial_indeg(self):
        e0, e1 = self.off[self.rb], self.off[self.re]
        return torch.as_tensor(np.bincount(self.tgt[e0:e1], minlength=self.n).astype(np.int32))

    def init(self, tid, ntid, indeg, norm0):
        n = self.n
        self.deg = indeg.numpy().astype(np.int64)
        s = [1.0 / n] * n  # scoring.cpp:96
        if tid is not None:
            w = n / ntid  # scoring.cpp:94-95
            for i in tid.tolist():
                s[i] = s[i] * w
        for j in range(n):
            norm0[j] = s[j] / max(int(self.deg[j]), 1)  # :59-61

    def step(self, damp, nin, nout, sout, rb, re, last):
        assert self.rb <= rb and re <= self.re
        base = (1.0 - damp) / self.n  # :53
        x = nin.tolist()
        for r in range(rb, re):
            acc = 0.0
            for w in self.tgt[self.off[r]:self.off[r + 1]]:
                acc += x[w]  # :66-68, in storage order
            nx = base + damp * acc  # :69 (two roundings, no FMA)
            if last:
                sout[r] = nx
            else:
                nout[r] = nx / max(int(self.deg[r]), 1)

    def sync(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, off, tgt, tid, iters, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blocks = D.edge_blocks(off, world)
        st = CpuStepper(off, tgt, blocks[rank])
        t = None if tid is None else torch.as_tensor(tid.astype(np.int64))
        out = D.reverse_pagerank_partitioned(st, len(off) - 1, iters, 0.85, t,
                                             0 if tid is None else len(tid), blocks=blocks)
        q.put((rank, out.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def _run(world, off, tgt, tid, iters):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, off, tgt, tid, iters, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_row_blocks_cover_and_pad():
    for n in (0, 1, 5, 31, 32, 1000, 1001):
        for world in (1, 2, 3, 8):
            chunk, blocks = D.row_blocks(n, world)
            assert chunk * world >= n and (n == 0 or chunk * world - n < world)
            rows = [r for b in blocks for r in range(*b)]
            assert rows == list(range(n))


def test_edge_blocks_cover_balance_and_match_the_library():
    """Edge-balanced blocks cover every row once, keep every block within one
    row's length of E/world, and equal the C-ABI's tg_row_blocks."""
    from paper_2111_05894_b200 import synth, tiergraph as tg
    port = oracle.port()
    cases = [port.from_edge_list(n, *(np.random.default_rng(n).integers(0, max(n, 1), (2, 6 * n))
                                      .astype(np.uint64))) for n in (1, 7, 100, 1001)]
    cases.append((np.zeros(6, np.uint64), np.zeros(0, np.uint64)))
    cases.append(synth.rmat_graph(200_000, 3_000_000, seed=2, device="cpu"))
    for off, tgt in cases:
        n, e = len(off) - 1, len(tgt)
        rowlen = np.diff(off.astype(np.int64))
        for world in (1, 2, 3, 8):
            blocks = D.edge_blocks(off, world)
            assert [r for b in blocks for r in range(*b)] == list(range(n))
            b = np.array([x[0] for x in blocks] + [n])
            assert np.array_equal(b.astype(np.uint64), tg.row_blocks(off, world))
            per = np.diff(off[b].astype(np.int64))
            if e:
                assert per.max() <= e / world + (rowlen.max() if n else 0) + 1
        if n > 100_000:  # R-MAT: near-equal edges per block
            for world in (2, 4, 8):
                b = tg.row_blocks(off, world).astype(np.int64)
                assert np.diff(off[b].astype(np.int64)).max() <= 1.1 * e / world


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_pagerank_over_gloo_is_bit_exact(world):
    port = oracle.port()
    chk = oracle.ref() or port
    n = 157
    rng = np.random.default_rng(world)
    src = np.concatenate([rng.integers(0, n, 900), np.zeros(120, np.int64)]).astype(np.uint64)
    dst = np.concatenate([rng.integers(0, n, 900), rng.integers(0, n, 120)]).astype(np.uint64)
    off, tgt = port.from_edge_list(n, src, dst)
    tid = port.draw_random_train_ids(n, 30, 7)
    for iters in (1, 5):
        res = _run(world, off, tgt, tid, iters)
        want = chk.weighted_reverse_pagerank(off, tgt, tid, iters, 0.85).tobytes()
        assert all(v == want for v in res.values()), f"world={world} iters={iters}"
    res = _run(world, off, tgt, None, 3)
    want = chk.reverse_pagerank(off, tgt, 3, 0.85).tobytes()
    assert all(v == want for v in res.values())


def _ipc_worker(rank, world, port, off, tgt, tid, q):
    """One process per rank, all on cuda:0 (the gpurun box has one GPU): the
    cross-process fused exchange (CUDA-IPC peer stores + device barrier)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_05894_b200 import tiergraph as tg
        ctx = tg.Context(0)
        g = tg.CsrGraph(off, tgt)
        ex = D.PeerExchangePagerank(g, ctx)
        outs = []
        for iters in (5, 1, 2):  # reuse of the shared vectors and counters across runs
            s = D.weighted_reverse_pagerank_ipc(g, tg.PagerankConfig(iters, 0.85), tid, ctx=ctx,
                                                exchange=ex)
            outs.append(s.cpu().numpy().tobytes())
        dist.barrier()
        ex.close()
        q.put((rank, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_across_processes_is_bit_exact(world):
    port = oracle.port()
    chk = oracle.ref() or port
    from paper_2111_05894_b200 import synth
    off, tgt = synth.rmat_graph(30_000, 400_000, seed=world)
    tid = port.draw_random_train_ids(len(off) - 1, 3_000, 5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p0 = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, p0, off, tgt, tid, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, iters in enumerate((5, 1, 2)):
        want = chk.weighted_reverse_pagerank(off, tgt, tid, iters, 0.85).tobytes()
        assert all(v[k] == want for v in res.values()), f"world={world} iters={iters}"


def _gather_worker(rank, world, port, n, dim, q):
    """One process per rank on cuda:0: the hot tier sharded over the ranks
    (interleaved rows, peer reads through CUDA-IPC mappings) and ONE cold tier
    for the node in POSIX shared memory (rank 0 fills it, the others map it)."""
    import ctypes as C
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_05894_b200 import synth, tiergraph as tg
        from paper_2111_05894_b200._lib import LIB
        chk = oracle.ref() or oracle.port()
        ctx = tg.Context(0)
        feat = synth.test_features(n, dim)
        perm = tg.NodePermutation(np.random.default_rng(3).permutation(n).astype(np.uint64))
        lay = tg.plan_layout(n, 0.3, 0.05, world, dim, 4)
        store = tg.TieredFeatureStore(None, None, lay, rank, ctx=ctx, place=False)
        name = f"/tg_test_cold_{port}"
        seg = tg.SharedHostSegment(name, store.cold_tier_bytes, create=(rank == 0))  \
            if rank == 0 else None
        dist.barrier()
        if rank != 0:
            seg = tg.SharedHostSegment(name, store.cold_tier_bytes, create=False)
        store.attach_cold(seg, fill=(rank == 0))
        if rank == 0:
            store.place(feat, perm)
        dist.barrier()  # the cold rows are in the segment
        if rank != 0:
            store.place(feat, perm)
        h = (C.c_uint8 * 64)()
        assert LIB.tg_ipc_get_handle(C.c_void_p(store.local_base), h) == 0
        allh = [None] * world
        dist.all_gather_object(allh, bytes(h))
        opened = []
        for d in range(world):
            if d == rank:
                continue
            p = C.c_void_p()
            assert LIB.tg_ipc_open_handle(ctx.h, (C.c_uint8 * 64).from_buffer_copy(allh[d]),
                                          C.byref(p)) == 0
            store.set_peer(d, p.value)
            opened.append(p.value)
        dist.barrier()
        inv = np.empty(n, np.uint64)
        inv[perm.new_id_of.astype(np.int64)] = np.arange(n, dtype=np.uint64)
        ok = True
        rng = np.random.default_rng(10 + rank)
        for _ in range(4):
            ids = np.unique(rng.integers(0, n, 3000)).astype(np.uint64)
            rep = tg.TrafficReport()
            got = store.gather_rows(ids, report=rep)
            ok &= bool(np.array_equal(got.view(np.float32), synth.expected_rows(inv[ids], dim)))
            ok &= bool(np.array_equal(rep.as_array(), chk.gather(lay.as_tuple(), ids, rank)))
            ok &= rep.peer_accesses > 0 and rep.host_accesses > 0
        dist.barrier()
        for p in opened:
            LIB.tg_ipc_close_handle(C.c_void_p(p))
        store.close()
        dist.barrier()
        seg.close()
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_ipc_gather_with_node_shared_cold_tier(world):
    """K8 across processes: rows byte-exact and TrafficReports equal to the
    reference gather() for every rank, with peer rows read over CUDA-IPC and
    one shared cold tier for the node."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p0 = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, p0, 40_000, 64, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res.values()), res
    assert not os.path.exists(f"/dev/shm/tg_test_cold_{p0}")
