"""Host-side producers of the hot path's inputs (not the hot path).

Thin bindings of csrc/host_producers.cpp — the reference's counter-based
train-id draw (scoring.cpp:22-31), transpose (csr_graph.cpp:67-80) and
GraphSAGE minibatch expansion (sampling.cpp:56-90, scheduled per epoch like
run_training_trace, sampling.cpp:106-123) — so the gather sees exactly the
reference's sampled node-id lists.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np

from ._lib import LIB
from .tiergraph import CsrGraph, DomainError, TierGraphError, TrainIdSet


def _host_check(rc: int):
    if rc != 0:
        msg = LIB.tg_host_last_error().decode(errors="replace")
        raise (DomainError if rc == 2 else TierGraphError)(msg)


def _take(p: C.c_void_p, n: int) -> np.ndarray:
    if n == 0:
        LIB.tg_free(p)
        return np.zeros(0, np.uint64)
    a = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), shape=(n,)).copy()
    LIB.tg_free(p)
    return a


def draw_random_train_ids(num_nodes: int, count: int, seed: int) -> TrainIdSet:
    """scoring.hpp:24 (scoring.cpp:22-31)"""
    out = np.empty(max(count, 1), np.uint64)
    _host_check(LIB.tg_draw_random_train_ids(int(num_nodes), int(count), int(seed), out.ctypes.data))
    return TrainIdSet(out[:count])


def transpose(g: CsrGraph) -> CsrGraph:
    """csr_graph.hpp:48 (csr_graph.cpp:67-80)"""
    off = np.ascontiguousarray(np.asarray(g.offsets, np.uint64))
    tgt = np.ascontiguousarray(np.asarray(g.targets, np.uint64))
    n = len(off) - 1
    t_off = np.empty(n + 1, np.uint64)
    t_tgt = np.empty(max(len(tgt), 1), np.uint64)
    _host_check(LIB.tg_transpose_host(off.ctypes.data, (tgt if len(tgt) else t_tgt).ctypes.data,
                                      n, t_off.ctypes.data, t_tgt.ctypes.data))
    return CsrGraph(t_off, t_tgt[:len(tgt)])


def epoch_minibatches(gt: CsrGraph, tid, fanouts: Sequence[int], batch_size: int, seed: int,
                      epoch: int, first_batch: int = 0, max_batches: int = 0,
                      threads: int = 0) -> List[np.ndarray]:
    """The sorted unique node-id list of each minibatch of one epoch, exactly
    as run_training_trace builds them (shuffle key {0x5348, epoch}; batch b
    expanded with BatchRng{seed, epoch, b}). `gt` is the TRANSPOSED graph."""
    ids = np.ascontiguousarray(np.asarray(tid.ids if isinstance(tid, TrainIdSet) else tid,
                                          np.uint64))
    f = np.ascontiguousarray(np.asarray(list(fanouts), np.uint32))
    off = np.ascontiguousarray(np.asarray(gt.offsets, np.uint64))
    tgt = np.ascontiguousarray(np.asarray(gt.targets, np.uint64))
    if len(tgt) == 0:
        tgt = np.zeros(1, np.uint64)
    po, nb, pi = C.c_void_p(), C.c_uint64(), C.c_void_p()
    _host_check(LIB.tg_epoch_minibatches(off.ctypes.data, tgt.ctypes.data, len(off) - 1,
                                         ids.ctypes.data, len(ids), f.ctypes.data, len(f),
                                         int(batch_size), int(seed), int(epoch), int(first_batch),
                                         int(max_batches), int(threads), C.byref(po), C.byref(nb),
                                         C.byref(pi)))
    o = _take(po, nb.value + 1)
    allids = _take(pi, int(o[-1]) if len(o) else 0)
    return [allids[o[b]:o[b + 1]] for b in range(nb.value)]


def epoch_order(tid, seed: int, epoch: int) -> np.ndarray:
    """sampling.cpp:106-109: this epoch's shuffled train ids; batch b is
    order[b*batch_size : (b+1)*batch_size]."""
    ids = np.ascontiguousarray(np.asarray(tid.ids if isinstance(tid, TrainIdSet) else tid,
                                          np.uint64))
    out = np.empty(max(len(ids), 1), np.uint64)
    _host_check(LIB.tg_epoch_order(ids.ctypes.data if len(ids) else out.ctypes.data, len(ids),
                                   int(seed), int(epoch), out.ctypes.data))
    return out[:len(ids)]


class TieredGraph:
    """Graph-structure tiering: the
    TRANSPOSED, score-reordered graph placed by `layout` for device
    `device_index` (csrc/structure.cu): rows [0, lb) and this device's
    interleaved slice of [lb, mb) in HBM, rows [mb, N) in pinned host memory
    (own, or `cold` = a mapped caller buffer / SharedHostSegment written by
    this graph when fill=True). Peers: set_peer(d, other.local_base) in one
    process, or the CUDA-IPC mapping of another process's local_base."""

    def __init__(self, offsets, targets, layout, device_index: int = 0, ctx=None, cold=None,
                 fill: bool = True):
        from . import tiergraph as tg
        self.tg = tg
        self.ctx = ctx or tg.default_context()
        off, tgt = tg._u64(offsets), tg._u64(targets)
        self.n = len(off) - 1
        self.e = len(tgt)
        self.layout = layout
        lay = layout._c() if hasattr(layout, "_c") else layout
        cptr, cbytes = None, 0
        if cold is not None:
            arr = cold.array if hasattr(cold, "array") else cold
            cptr, cbytes = tg._ptr(arr), int(arr.nbytes)
        h = C.c_void_p()
        tg._check(LIB.tg_sgraph_create(self.ctx.h, C.byref(lay), int(device_index), tg._ptr(off),
                                       tg._nonempty(tgt, np.uint64), self.n, self.e, cptr, cbytes,
                                       int(bool(fill)), C.byref(h)))
        self.h = h
        self.device_index = int(device_index)

    @staticmethod
    def cold_bytes(offsets, layout) -> int:
        from . import tiergraph as tg
        off = tg._u64(offsets)
        lay = layout._c() if hasattr(layout, "_c") else layout
        return int(LIB.tg_sgraph_cold_bytes(tg._ptr(off), len(off) - 1, C.byref(lay)))

    @property
    def local_base(self) -> int:
        return LIB.tg_sgraph_local_base(self.h) or 0

    @property
    def cold_host(self) -> int:
        return LIB.tg_sgraph_cold_host(self.h) or 0

    def set_peer(self, d: int, base: int) -> None:
        self.tg._check(LIB.tg_sgraph_set_peer(self.h, int(d), C.c_void_p(base)))

    def info(self) -> dict:
        out = np.zeros(4, np.uint64)
        self.tg._check(LIB.tg_sgraph_info(self.h, out.ctypes.data))
        return {"replicated_bytes": int(out[0]), "slice_bytes": int(out[1]),
                "host_bytes": int(out[2]), "offsets_bytes": int(out[3])}

    def close(self):
        if getattr(self, "h", None):
            LIB.tg_sgraph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GpuSampler:
    """build_minibatch (sampling.cpp:56-90) on the GPU, bit-identical member
    lists (csrc/sampling.cu). `gt` is the TRANSPOSED graph (producers.transpose)."""

    def __init__(self, gt, ctx=None):
        """gt: a CsrGraph (the whole transposed graph on this device) or a
        TieredGraph (its rows placed by a TierLayout)."""
        from . import tiergraph as tg
        self.tg = tg
        self.gt = gt
        h = C.c_void_p()
        if isinstance(gt, TieredGraph):
            self.ctx = ctx or gt.ctx
            self.n = gt.n
            tg._check(LIB.tg_sampler_create_tiered(self.ctx.h, gt.h, C.byref(h)))
        else:
            self.ctx = ctx or tg.default_context()
            self.n = gt.num_nodes()
            tg._check(LIB.tg_sampler_create(self.ctx.h, gt.device(self.ctx), C.byref(h)))
        self.h = h
        self._pinned = None  # reusable pinned output (members of one minibatch)

    def _out_buffer(self, ns: int, fanouts) -> np.ndarray:
        bound, layer = ns, ns
        for f in fanouts:
            layer = min(self.n, layer * int(f))
            bound += layer
        bound = max(1, min(bound, self.n))
        if self._pinned is None or len(self._pinned) < bound:
            self._pinned = self.tg.host_alloc(8 * bound).view(np.uint64)
        return self._pinned

    def minibatch(self, seeds, fanouts: Sequence[int], seed: int, epoch: int, batch: int,
                  out=None):
        """Sorted unique member ids (numpy u64, or into a device tensor `out`,
        returning the member count)."""
        tg = self.tg
        sd = tg._u64(seeds)
        fo = np.ascontiguousarray(np.asarray(list(fanouts), np.uint32))
        cnt = C.c_uint64()
        dst = out if out is not None else self._out_buffer(len(sd), fanouts)
        tg._check(LIB.tg_sample_minibatch(self.h, tg._nonempty(sd, np.uint64), tg._len(sd),
                                          fo.ctypes.data if len(fo) else None, len(fo),
                                          int(seed), int(epoch), int(batch), tg._ptr(dst),
                                          tg._len(dst), C.byref(cnt)))
        return int(cnt.value) if out is not None else dst[:cnt.value].copy()

    def batches(self, order, fanouts: Sequence[int], batch_size: int, seed: int, epoch: int,
                first_batch: int = 0, nbatches: int = None, device: bool = False):
        """Member lists of batches [first_batch, first_batch + nbatches) of an
        epoch whose shuffled train ids are `order` (epoch_order), expanded on
        the device back to back with one host round trip in total. With
        device=True returns (the concatenated member lists as a CUDA int64
        tensor, the u64 offsets) without copying them to the host; the tensor
        is reused by the next call."""
        tg = self.tg
        od = tg._u64(order)
        nb_all = (len(od) + batch_size - 1) // batch_size
        if nbatches is None:
            nbatches = nb_all - first_batch
        fo = np.ascontiguousarray(np.asarray(list(fanouts), np.uint32))
        per, layer = batch_size, batch_size
        for f in fanouts:
            layer = min(self.n, layer * int(f))
            per += layer
        cap = max(1, nbatches * min(per, self.n))
        md = self._device_buffer(cap)
        offs = np.empty(nbatches + 1, np.uint64)
        tg._check(LIB.tg_sample_batches(self.h, tg._nonempty(od, np.uint64), len(od), batch_size,
                                        first_batch, nbatches,
                                        fo.ctypes.data if len(fo) else None, len(fo), int(seed),
                                        int(epoch), md.data_ptr(), cap, offs.ctypes.data))
        if device:
            return md, offs
        total = int(offs[-1])
        host = self._host_buffer(total)
        host_t = self._torch.from_numpy(host[:total].view(np.int64))
        host_t.copy_(md[:total])  # pinned: one DMA
        allm = host[:total].copy()
        return [allm[int(offs[k]):int(offs[k + 1])] for k in range(nbatches)]

    def _device_buffer(self, cap: int):
        import torch
        self._torch = torch
        if getattr(self, "_dbuf", None) is None or self._dbuf.numel() < cap:
            self._dbuf = torch.empty(cap, dtype=torch.int64,
                                     device=torch.device("cuda", self.ctx.device))
        return self._dbuf

    def _host_buffer(self, n: int) -> np.ndarray:
        if getattr(self, "_hbuf", None) is None or len(self._hbuf) < n:
            self._hbuf = self.tg.host_alloc(8 * max(n, 1)).view(np.uint64)
        return self._hbuf

    def minibatch_raw(self, seeds, fanouts: Sequence[int], seed: int, epoch: int, batch: int):
        """(members, raw draws) — build_minibatch with raw_draws (sampling.hpp:48-55);
        the raw draws come back sorted (their order is unspecified)."""
        tg = self.tg
        sd = tg._u64(seeds)
        fo = np.ascontiguousarray(np.asarray(list(fanouts), np.uint32))
        cap = self.n
        raw_cap = len(sd) + sum(int(f) for f in fanouts) * self.n
        raw_cap = min(raw_cap, 1 << 24)
        out = np.empty(max(cap, 1), np.uint64)
        raw = np.empty(max(raw_cap, 1), np.uint64)
        cnt, rn = C.c_uint64(), C.c_uint64()
        tg._check(LIB.tg_sample_minibatch_raw(self.h, tg._nonempty(sd, np.uint64), tg._len(sd),
                                              fo.ctypes.data if len(fo) else None, len(fo),
                                              int(seed), int(epoch), int(batch), out.ctypes.data,
                                              cap, C.byref(cnt), raw.ctypes.data, raw_cap,
                                              C.byref(rn)))
        return out[:cnt.value].copy(), np.sort(raw[:rn.value])

    def trace(self, tid, fanouts: Sequence[int], batch_size: int, epochs: int, seed: int,
              dedup_per_batch: bool = True, out=None):
        """run_training_trace (sampling.cpp:92-140) on the device: per-node
        access counts (numpy u64, or into the device tensor `out`)."""
        tg = self.tg
        ids = tg._u64(tid.ids if isinstance(tid, TrainIdSet) else tid)
        fo = np.ascontiguousarray(np.asarray(list(fanouts), np.uint32))
        dst = out if out is not None else np.empty(max(self.n, 1), np.uint64)
        tg._check(LIB.tg_sampler_trace(self.h, tg._nonempty(ids, np.uint64), tg._len(ids),
                                       fo.ctypes.data if len(fo) else None, len(fo),
                                       int(batch_size), int(epochs), int(seed),
                                       int(bool(dedup_per_batch)), tg._ptr(dst)))
        return dst if out is not None else dst[:self.n]

    def structure_reads(self, reset: bool = False) -> np.ndarray:
        """Neighbour ids read per tier {local HBM, peer HBM, host} since the
        last reset (a sampler over a TieredGraph only)."""
        out = np.zeros(3, np.uint64)
        self.tg._check(LIB.tg_sampler_structure_reads(self.h, out.ctypes.data, int(reset)))
        return out

    def close(self):
        if getattr(self, "h", None):
            LIB.tg_sampler_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
