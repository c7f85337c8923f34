"""Python host mirror of the reference `tiergraph` hot-path API, on the B200.

Same names, argument meaning and error behaviour as the reference C++ API
(proj/include/tiergraph/{scoring,reorder,tiering}.hpp), so a test written
against the reference reads the same here. Every computation runs in
libtiergraph_b200.so through the C-ABI (include/tg_capi.h); this module only
marshals arrays. Arrays may be numpy (host) or torch CUDA tensors (device);
results come back as numpy unless an `out=` array/tensor is given.

Reference exceptions map to DomainError / FormatError / IoError
(types.hpp:13-29); CUDA failures raise TierGraphError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Iterable, Optional, Sequence

import numpy as np

from ._lib import (LIB, TG_COLD_INDIRECT, TG_COLD_PAD128, TG_COLD_REORDERED, TG_COLD_SPLIT_TAIL,
                   TG_GATHER_BULK, TG_GATHER_DYNAMIC,
                   TG_GATHER_L2PF, TG_GATHER_SPREAD, TgLayout, TgLocation, TgReport)

__all__ = [
    "TierGraphError", "DomainError", "FormatError", "IoError", "Context", "default_context",
    "CsrGraph", "FeatureMatrix", "TrainIdSet", "PagerankConfig", "NodePermutation", "TierLayout",
    "Tier", "Location", "LinkCostModel", "TrafficReport", "SweepRow", "AccessCounter",
    "degree_score", "in_degrees", "reverse_pagerank", "weighted_reverse_pagerank",
    "score_ordering", "permutation_from_scores", "validate_permutation", "invert",
    "reorder_graph", "reorder_features", "validate_layout", "validate_cost_model", "resolve",
    "plan_layout", "gather", "simulate_trace", "counts_in_row_order", "hot_fraction_sweep",
    "make_access_counter", "TieredFeatureStore", "kernel_launches",
]


# ------------------------------------------------------------------ errors
class TierGraphError(RuntimeError):
    """A CUDA / internal failure (reference CLI exit code 5)."""


class DomainError(TierGraphError, ValueError):
    """Reference DomainError (types.hpp:26-29): a precondition was violated."""


class FormatError(TierGraphError):
    """Reference FormatError (types.hpp:20-23)."""


class IoError(TierGraphError, OSError):
    """Reference IoError (types.hpp:13-16)."""


_ERR = {2: DomainError, 3: FormatError, 4: IoError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = LIB.tg_last_error().decode(errors="replace")
        raise _ERR.get(rc, TierGraphError)(msg)


def kernel_launches() -> int:
    """Kernels this process launched through libtiergraph_b200 so far."""
    return int(LIB.tg_kernel_launches())


# ------------------------------------------------------------------ arrays
def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if _is_torch(a):
        if not a.is_contiguous():
            raise DomainError("tensor must be contiguous")
        return a.data_ptr() or None
    if not a.flags["C_CONTIGUOUS"]:
        raise DomainError("array must be C-contiguous")
    return a.ctypes.data or None


def _len(a) -> int:
    return int(a.numel()) if _is_torch(a) else int(a.size)


def _as(a, np_dtype, torch_name: str):
    """numpy arrays are converted (copy if needed); torch tensors must match."""
    if _is_torch(a):
        import torch
        want = getattr(torch, torch_name)
        if a.dtype != want:
            a = a.to(want)
        return a.contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np_dtype))


def _u64(a):
    return _as(a, np.uint64, "uint64")


def _f64(a):
    return _as(a, np.float64, "float64")


def _nbytes(a) -> int:
    return int(a.numel() * a.element_size()) if _is_torch(a) else int(a.nbytes)


def _check_out(out, need: int, what: str = "out"):
    """A caller output buffer must be contiguous and hold `need` bytes (the
    library writes exactly that many and cannot see the buffer's size)."""
    _ptr(out)  # contiguity
    if _nbytes(out) < need:
        raise DomainError(f"{what} holds {_nbytes(out)} bytes, {need} needed")


def _nonempty(a, dtype):
    """Pointer for a possibly empty array (the C side never dereferences it)."""
    if _len(a) == 0:
        return np.zeros(1, dtype).ctypes.data
    return _ptr(a)


# ---------------------------------------------------------------- context
class Context:
    """One device + stream (tg_ctx). `stream` may be a torch.cuda.Stream to
    run stream-ordered with torch work."""

    def __init__(self, device: Optional[int] = None, stream=None):
        if device is None:
            device = int(LIB.tg_default_device())
        h = C.c_void_p()
        if stream is not None:
            _check(LIB.tg_ctx_create_on_stream(device, C.c_void_p(stream.cuda_stream), C.byref(h)))
        else:
            _check(LIB.tg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def sync(self):
        _check(LIB.tg_ctx_sync(self.h))

    def trim(self):
        """Free the context's scratch and the device pool's cached memory."""
        _check(LIB.tg_ctx_trim(self.h))

    @property
    def stream_ptr(self) -> int:
        return int(LIB.tg_ctx_stream(self.h) or 0)

    def close(self):
        if getattr(self, "h", None):
            LIB.tg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT: Optional[Context] = None


def default_context() -> Context:
    """Process-wide context on TIERGRAPH_DEVICES' first device (parallel.cpp:13-19)."""
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context()
    return _DEFAULT


# ------------------------------------------------------------ data types
class DeviceCsrGraph:
    """A CsrGraph that exists only on the device (tg_graph_load_csrg): the
    same calls accept it wherever they take a CsrGraph bound to `ctx`."""

    def __init__(self, ctx: "Context", h):
        self._ctx, self._h = ctx, h

    def num_nodes(self) -> int:
        return int(LIB.tg_graph_num_nodes(self._h))

    def num_edges(self) -> int:
        return int(LIB.tg_graph_num_edges(self._h))

    def device(self, ctx: "Context"):
        if ctx is not self._ctx:
            raise DomainError("this graph lives on another context")
        return self._h

    def release(self):
        if self._h:
            LIB.tg_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def load_csr_device(path, *, ctx: "Context" = None) -> DeviceCsrGraph:
    """io.hpp:26 load_csr, straight into the device layout (CSRG v1)."""
    c = _ctx(ctx)
    h = C.c_void_p()
    _check(LIB.tg_graph_load_csrg(c.h, str(path).encode(), C.byref(h)))
    return DeviceCsrGraph(c, h)


class CsrGraph:
    """csr_graph.hpp:22-35. Row u = targets[offsets[u]:offsets[u+1]] (out-neighbors).

    The device copy (u32 CSR + row-group schedule) is built on first use and
    cached per context; treat the arrays as immutable afterwards.
    """

    def __init__(self, offsets, targets):
        self.offsets = _u64(offsets)
        self.targets = _u64(targets)
        self._dev = {}

    def num_nodes(self) -> int:
        return max(_len(self.offsets) - 1, 0)

    def num_edges(self) -> int:
        return _len(self.targets)

    def row(self, u):
        return self.targets[int(self.offsets[u]):int(self.offsets[u + 1])]

    def out_degree(self, u) -> int:
        return int(self.offsets[u + 1] - self.offsets[u])

    def device(self, ctx: Context):
        key = id(ctx)
        if key not in self._dev:
            h = C.c_void_p()
            if _len(self.offsets) == 0:
                raise FormatError("csr: offsets array is empty")
            _check(LIB.tg_graph_create(ctx.h, _ptr(self.offsets), _nonempty(self.targets, np.uint64),
                                       self.num_nodes(), self.num_edges(), C.byref(h)))
            self._dev[key] = (ctx, h)
        return self._dev[key][1]

    def release(self):
        for ctx, h in self._dev.values():
            LIB.tg_graph_destroy(h)
        self._dev.clear()

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    def __eq__(self, other):
        return (np.array_equal(np.asarray(self.offsets), np.asarray(other.offsets))
                and np.array_equal(np.asarray(self.targets), np.asarray(other.targets)))


@dataclasses.dataclass
class FeatureMatrix:
    """feature_matrix.hpp:14-28: row-major rows of opaque fixed-width elements."""
    num_rows: int
    dim: int
    elem_bytes: int
    data: np.ndarray  # uint8 [num_rows * dim * elem_bytes] (or any dtype viewable as bytes)

    def row_bytes(self) -> int:
        return self.dim * self.elem_bytes

    def row(self, r):
        rb = self.row_bytes()
        return self.data.reshape(-1).view(np.uint8)[r * rb:(r + 1) * rb]

    @staticmethod
    def from_array(a: np.ndarray) -> "FeatureMatrix":
        a = np.ascontiguousarray(a)
        rows = a.shape[0]
        dim = int(np.prod(a.shape[1:])) if a.ndim > 1 else 1
        return FeatureMatrix(rows, dim, a.dtype.itemsize, a.reshape(-1).view(np.uint8))


@dataclasses.dataclass
class TrainIdSet:
    """scoring.hpp:15-20. Sorted unique ids of labeled nodes."""
    ids: np.ndarray

    @staticmethod
    def from_ids(raw, num_nodes: int) -> "TrainIdSet":  # scoring.cpp:13-20
        ids = np.unique(np.asarray(raw, dtype=np.uint64))
        if ids.size and int(ids[-1]) >= num_nodes:
            raise DomainError(f"train id {int(ids[-1])} out of range for num_nodes={num_nodes}")
        return TrainIdSet(ids)


@dataclasses.dataclass
class PagerankConfig:
    """scoring.hpp:26-29"""
    iterations: int = 5
    damp: float = 0.85


@dataclasses.dataclass
class NodePermutation:
    """reorder.hpp:13-18: old node id -> new node id."""
    new_id_of: np.ndarray

    def size(self) -> int:
        return _len(self.new_id_of)

    def __getitem__(self, old):
        return self.new_id_of[old]


class Tier:
    LocalHot = 0
    InterleavedDevice = 1
    ColdHost = 2


@dataclasses.dataclass(frozen=True)
class Location:
    """tiering.hpp:31-37"""
    tier: int = Tier.ColdHost
    device: int = 0
    row_within_tier: int = 0


@dataclasses.dataclass
class TierLayout:
    """tiering.hpp:16-25"""
    num_rows: int = 0
    local_boundary: int = 0
    multi_boundary: int = 0
    num_devices: int = 1
    feature_dim: int = 0
    elem_bytes: int = 0

    def bytes_per_row(self) -> int:
        return self.feature_dim * self.elem_bytes

    def as_tuple(self):
        return (self.num_rows, self.local_boundary, self.multi_boundary, self.num_devices,
                self.feature_dim, self.elem_bytes)

    def _c(self) -> TgLayout:
        return TgLayout(*self.as_tuple())

    @staticmethod
    def _from_c(l: TgLayout) -> "TierLayout":
        return TierLayout(l.num_rows, l.local_boundary, l.multi_boundary, l.num_devices,
                          l.feature_dim, l.elem_bytes)


@dataclasses.dataclass
class LinkCostModel:
    """tiering.hpp:40-44 (GB/s)"""
    local_gbps: float = 900.0
    peer_gbps: float = 150.0
    host_gbps: float = 16.0


_REPORT_FIELDS = ("local_accesses", "peer_accesses", "host_accesses", "local_bytes",
                  "peer_bytes", "host_bytes")


@dataclasses.dataclass
class TrafficReport:
    """tiering.hpp:51-68"""
    local_accesses: int = 0
    peer_accesses: int = 0
    host_accesses: int = 0
    local_bytes: int = 0
    peer_bytes: int = 0
    host_bytes: int = 0

    def total_accesses(self) -> int:
        return self.local_accesses + self.peer_accesses + self.host_accesses

    def hit_ratio(self) -> float:
        return float(LIB.tg_report_hit_ratio(C.byref(self._c())))

    def est_transfer_seconds(self, cost: LinkCostModel = LinkCostModel()) -> float:
        return float(LIB.tg_report_est_transfer_seconds(C.byref(self._c()), cost.local_gbps,
                                                        cost.peer_gbps, cost.host_gbps))

    def __iadd__(self, o: "TrafficReport"):
        for f in _REPORT_FIELDS:
            setattr(self, f, getattr(self, f) + getattr(o, f))
        return self

    def as_array(self) -> np.ndarray:
        return np.array([getattr(self, f) for f in _REPORT_FIELDS], np.uint64)

    def _c(self) -> TgReport:
        return TgReport(*[getattr(self, f) for f in _REPORT_FIELDS])

    def _load(self, r: TgReport):
        for f in _REPORT_FIELDS:
            setattr(self, f, int(getattr(r, f)))
        return self


@dataclasses.dataclass
class AccessCounter:
    """sampling.hpp:31-34"""
    counts: np.ndarray
    total: int = 0


def make_access_counter(counts) -> AccessCounter:  # sampling.cpp:27-33
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    return AccessCounter(c, int(c.sum(dtype=np.uint64)) if c.size else 0)


@dataclasses.dataclass
class SweepRow:
    """tiering.hpp:101-106"""
    hot_fraction: float
    replicated_fraction: float
    layout: TierLayout
    report: TrafficReport


# ------------------------------------------------------------- helpers
def _ctx(ctx: Optional[Context]) -> Context:
    return ctx or default_context()


def _out(out, n: int, np_dtype, torch_name: str):
    if out is None:
        return np.empty(n, np_dtype)
    if _len(out) != n:
        raise DomainError(f"out has {_len(out)} elements, need {n}")
    return out


def _ids(tid) -> object:
    if isinstance(tid, TrainIdSet):
        return _u64(tid.ids)
    return _u64(tid)


# ------------------------------------------------------------- scoring
def degree_score(g: CsrGraph, *, ctx: Context = None, out=None):
    """scoring.hpp:32 (scoring.cpp:33-38)"""
    c = _ctx(ctx)
    o = _out(out, g.num_nodes(), np.float64, "float64")
    if g.num_nodes():
        _check(LIB.tg_degree_score(c.h, g.device(c), _ptr(o)))
    return o


def in_degrees(g: CsrGraph, *, ctx: Context = None, out=None):
    """csr_graph.hpp:51 (csr_graph.cpp:89-93)"""
    c = _ctx(ctx)
    o = _out(out, g.num_nodes(), np.uint64, "uint64")
    if g.num_nodes():
        _check(LIB.tg_in_degrees(c.h, g.device(c), _ptr(o)))
    return o


def reverse_pagerank(g: CsrGraph, cfg: PagerankConfig = PagerankConfig(), *, ctx: Context = None,
                     out=None):
    """scoring.hpp:40 (scoring.cpp:78-84). Bit-identical to the reference."""
    c = _ctx(ctx)
    o = _out(out, g.num_nodes(), np.float64, "float64")
    gh = g.device(c) if g.num_nodes() else None
    _check(LIB.tg_reverse_pagerank(c.h, gh, cfg.iterations, cfg.damp, _ptr(o)))
    return o


def weighted_reverse_pagerank(g: CsrGraph, cfg: PagerankConfig = PagerankConfig(),
                              tid: TrainIdSet = None, *, ctx: Context = None, out=None):
    """scoring.hpp:45-46 (scoring.cpp:86-102). Bit-identical to the reference."""
    c = _ctx(ctx)
    ids = _ids(tid if tid is not None else np.zeros(0, np.uint64))
    o = _out(out, g.num_nodes(), np.float64, "float64")
    gh = g.device(c) if g.num_nodes() else None
    _check(LIB.tg_weighted_reverse_pagerank(c.h, gh, cfg.iterations, cfg.damp,
                                            _nonempty(ids, np.uint64), _len(ids), _ptr(o)))
    return o


def row_blocks(offsets, parts: int) -> np.ndarray:
    """Edge-balanced contiguous row blocks (tg_row_blocks): parts+1 bounds."""
    off = _u64(offsets)
    b = np.zeros(parts + 1, np.uint64)
    _check(LIB.tg_row_blocks(_ptr(off), max(_len(off) - 1, 0), parts, b.ctypes.data))
    return b


class MultiDeviceGraph:
    """A CsrGraph partitioned over several devices of this process
    (tg_mgraph): one edge-balanced row block per context, K1
    sharded and summed once, K3 steps exchanging the blocks by contiguous peer
    copies. PageRank is bit-identical to one device for any device count --
    what the C++ drop-in runs when TIERGRAPH_DEVICES lists several devices."""

    def __init__(self, g: CsrGraph, ctxs):
        self.ctxs = list(ctxs)
        self.n, self.e = g.num_nodes(), g.num_edges()
        arr = (C.c_void_p * len(self.ctxs))(*[c.h.value for c in self.ctxs])
        h = C.c_void_p()
        if _len(g.offsets) == 0:
            raise FormatError("csr: offsets array is empty")
        _check(LIB.tg_mgraph_create(arr, len(self.ctxs), _ptr(g.offsets),
                                    _nonempty(g.targets, np.uint64), self.n, self.e, C.byref(h)))
        self.h = h

    def info(self):
        G = len(self.ctxs)
        b = np.zeros(G + 1, np.uint64)
        e = np.zeros(G, np.uint64)
        ms = C.c_double()
        _check(LIB.tg_mgraph_info(self.h, b.ctypes.data, e.ctypes.data, C.byref(ms)))
        return {"bounds": b, "edges": e, "indeg_ms": ms.value}

    def in_degrees(self):
        o = np.empty(self.n, np.uint64)
        if self.n:
            _check(LIB.tg_mgraph_in_degrees(self.h, o.ctypes.data))
        return o

    def weighted_reverse_pagerank(self, cfg: PagerankConfig = PagerankConfig(),
                                  tid: TrainIdSet = None, out=None):
        ids = _ids(tid if tid is not None else np.zeros(0, np.uint64))
        o = _out(out, self.n, np.float64, "float64")
        _check(LIB.tg_mgraph_pagerank(self.h, cfg.iterations, cfg.damp,
                                      _nonempty(ids, np.uint64), _len(ids), 1, _ptr(o)))
        return o

    def reverse_pagerank(self, cfg: PagerankConfig = PagerankConfig(), out=None):
        o = _out(out, self.n, np.float64, "float64")
        _check(LIB.tg_mgraph_pagerank(self.h, cfg.iterations, cfg.damp, None, 0, 0, _ptr(o)))
        return o

    def close(self):
        if getattr(self, "h", None):
            LIB.tg_mgraph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def score_ordering(scores, *, ctx: Context = None, out=None):
    """scoring.hpp:49 (scoring.cpp:104-115)"""
    c = _ctx(ctx)
    s = _f64(scores)
    o = _out(out, _len(s), np.uint64, "uint64")
    if _len(s):
        _check(LIB.tg_score_ordering(c.h, _ptr(s), _len(s), _ptr(o)))
    return o


# ------------------------------------------------------------- reorder
def permutation_from_scores(scores, *, ctx: Context = None, out=None, order_out=None) -> NodePermutation:
    """reorder.hpp:25 (reorder.cpp:23-29)"""
    c = _ctx(ctx)
    s = _f64(scores)
    o = _out(out, _len(s), np.uint64, "uint64")
    if _len(s):
        _check(LIB.tg_permutation_from_scores(c.h, _ptr(s), _len(s), _ptr(o), _ptr(order_out)))
    return NodePermutation(o)


def _perm(p):
    return _u64(p.new_id_of if isinstance(p, NodePermutation) else p)


def validate_permutation(perm, *, ctx: Context = None) -> None:
    """reorder.hpp:21 (reorder.cpp:10-21)"""
    c = _ctx(ctx)
    p = _perm(perm)
    if _len(p):
        _check(LIB.tg_validate_permutation(c.h, _ptr(p), _len(p)))


def invert(perm, *, ctx: Context = None) -> NodePermutation:
    """reorder.hpp:27 (reorder.cpp:31-37)"""
    c = _ctx(ctx)
    p = _perm(perm)
    o = np.empty(_len(p), np.uint64)
    if _len(p):
        _check(LIB.tg_invert(c.h, _ptr(p), _len(p), _ptr(o)))
    return NodePermutation(o)


def reorder_graph(g: CsrGraph, perm, *, ctx: Context = None) -> CsrGraph:
    """reorder.hpp:33 (reorder.cpp:39-66)"""
    c = _ctx(ctx)
    p = _perm(perm)
    n, e = g.num_nodes(), g.num_edges()
    oo = np.empty(n + 1, np.uint64)
    ot = np.empty(max(e, 1), np.uint64)
    _check(LIB.tg_reorder_graph(c.h, _ptr(g.offsets), _nonempty(g.targets, np.uint64), n, e,
                                _nonempty(p, np.uint64), _len(p), _ptr(oo), _ptr(ot)))
    return CsrGraph(oo, ot[:e])


def transpose(g: CsrGraph, *, ctx: Context = None) -> CsrGraph:
    """csr_graph.hpp:48 (csr_graph.cpp:67-80), on the device."""
    c = _ctx(ctx)
    n, e = g.num_nodes(), g.num_edges()
    oo = np.empty(n + 1, np.uint64)
    ot = np.empty(max(e, 1), np.uint64)
    _check(LIB.tg_transpose(c.h, _ptr(g.offsets), _nonempty(g.targets, np.uint64), n, e, _ptr(oo),
                            _ptr(ot)))
    return CsrGraph(oo, ot[:e])


def reorder_features(f: FeatureMatrix, perm, *, ctx: Context = None) -> FeatureMatrix:
    """reorder.hpp:40 (reorder.cpp:97-117): new row perm[u] = old row u."""
    c = _ctx(ctx)
    p = _perm(perm)
    data = np.ascontiguousarray(f.data).reshape(-1).view(np.uint8)
    want = f.num_rows * f.dim * f.elem_bytes
    if data.size != want:  # feature_matrix.cpp:9-14
        raise FormatError(f"features: data holds {data.size} bytes, expected {want}")
    out = np.empty_like(data)
    _check(LIB.tg_reorder_features(c.h, _nonempty(data, np.uint8), f.num_rows, f.row_bytes(),
                                   _nonempty(p, np.uint64), _len(p), _nonempty(out, np.uint8)))
    return FeatureMatrix(f.num_rows, f.dim, f.elem_bytes, out)


# ------------------------------------------------------------- tiering
def validate_layout(layout: TierLayout) -> None:
    _check(LIB.tg_validate_layout(C.byref(layout._c())))


def validate_cost_model(cost: LinkCostModel) -> None:
    _check(LIB.tg_validate_cost_model(cost.local_gbps, cost.peer_gbps, cost.host_gbps))


def resolve(layout: TierLayout, row_id: int, requesting_device: int) -> Location:
    """tiering.hpp:74-75 (tiering.cpp:48-65)"""
    loc = TgLocation()
    _check(LIB.tg_resolve(C.byref(layout._c()), int(row_id), int(requesting_device), C.byref(loc)))
    return Location(int(loc.tier), int(loc.device), int(loc.row_within_tier))


def plan_layout(num_rows, hot_fraction, replicated_fraction, num_devices, feature_dim, elem_bytes,
                per_device_budget_bytes=0) -> TierLayout:
    """tiering.hpp:81-84 (tiering.cpp:67-98)"""
    l = TgLayout()
    _check(LIB.tg_plan_layout(int(num_rows), float(hot_fraction), float(replicated_fraction),
                              int(num_devices), int(feature_dim), int(elem_bytes),
                              int(per_device_budget_bytes), C.byref(l)))
    return TierLayout._from_c(l)


def gather(layout: TierLayout, row_ids, requesting_device: int, report: TrafficReport, *,
           ctx: Context = None) -> None:
    """tiering.hpp:88-89 (tiering.cpp:100-125): accounting only, accumulated into
    `report` (ids before an invalid one stay accounted, as in the reference)."""
    c = _ctx(ctx)
    ids = _u64(row_ids)
    r = report._c()
    try:
        _check(LIB.tg_gather_account(c.h, C.byref(layout._c()), _nonempty(ids, np.uint64),
                                     _len(ids), int(requesting_device), C.byref(r)))
    finally:
        report._load(r)


def simulate_trace(counter: AccessCounter, layout: TierLayout, *, ctx: Context = None) -> TrafficReport:
    """tiering.hpp:95 (tiering.cpp:127-162)"""
    c = _ctx(ctx)
    counts = _u64(counter.counts)
    r = TgReport()
    _check(LIB.tg_simulate_trace(c.h, _nonempty(counts, np.uint64), _len(counts),
                                 C.byref(layout._c()), C.byref(r)))
    return TrafficReport()._load(r)


def counts_in_row_order(counter: AccessCounter, ordering, *, ctx: Context = None):
    """tiering.hpp:98-99 (tiering.cpp:164-175)"""
    c = _ctx(ctx)
    counts = _u64(counter.counts)
    o = _u64(ordering)
    out = np.empty(_len(o), np.uint64)
    _check(LIB.tg_counts_in_row_order(c.h, _nonempty(counts, np.uint64), _len(counts),
                                      _nonempty(o, np.uint64), _len(o), _nonempty(out, np.uint64)))
    return out


def hot_fraction_sweep(counter: AccessCounter, ordering, fractions: Sequence[float],
                       replicated_fraction: float, num_devices: int, feature_dim: int,
                       elem_bytes: int, per_device_budget_bytes: int = 0, *,
                       ctx: Context = None):
    """tiering.hpp:110-117 (tiering.cpp:177-202)"""
    c = _ctx(ctx)
    counts = _u64(counter.counts)
    o = _u64(ordering)
    if _len(o) != _len(counts):
        raise DomainError("ordering length != counter length")
    fr = np.ascontiguousarray(np.asarray(list(fractions), np.float64))
    nf = len(fr)
    lays = (TgLayout * max(nf, 1))()
    reps = (TgReport * max(nf, 1))()
    rf = np.zeros(max(nf, 1), np.float64)
    _check(LIB.tg_hot_fraction_sweep(c.h, _nonempty(counts, np.uint64), _len(counts),
                                     _nonempty(o, np.uint64), _nonempty(fr, np.float64), nf,
                                     float(replicated_fraction), int(num_devices),
                                     int(feature_dim), int(elem_bytes),
                                     int(per_device_budget_bytes), lays, reps, rf.ctypes.data))
    return [SweepRow(float(fr[i]), float(rf[i]), TierLayout._from_c(lays[i]),
                     TrafficReport()._load(reps[i])) for i in range(nf)]


# ------------------------------------------------- tiered feature store
class TieredFeatureStore:
    """The byte-moving tiered gather (Listing 1) behind the
    reference's address map (tiering.cpp:48-65) and accounting (:100-125).

    One store per device: replicated rows [0, lb) and this device's
    interleaved slice of [lb, mb) live in its HBM; cold rows [mb, N) in pinned
    mapped host memory. Row ids are NEW ids (after the permutation).
    """

    def __init__(self, features, perm, layout: TierLayout, device_index: int = 0, *,
                 ctx: Context = None, cold_mode: str = "reordered", pad128: bool = True,
                 split_tail: bool = True, gather_mode: str = "bulk+spread+dynamic",
                 place: bool = True):
        self.ctx = _ctx(ctx)
        self.layout = layout
        self.device_index = device_index
        flags = {"reordered": TG_COLD_REORDERED, "indirect": TG_COLD_INDIRECT}[cold_mode]
        if pad128:
            flags |= TG_COLD_PAD128
        if split_tail:  # whole 128 B lines of each cold row in host memory, the rest in HBM
            flags |= TG_COLD_SPLIT_TAIL
        # gather_mode: "ldg" | "bulk" | "l2pf", optionally "+spread"
        for tok in gather_mode.split("+"):
            flags |= {"ldg": 0, "bulk": TG_GATHER_BULK, "l2pf": TG_GATHER_L2PF,
                      "spread": TG_GATHER_SPREAD, "dynamic": TG_GATHER_DYNAMIC}[tok]
        h = C.c_void_p()
        _check(LIB.tg_store_create(self.ctx.h, C.byref(layout._c()), int(device_index), flags,
                                   C.byref(h)))
        self.h = h
        self._keep = []
        if place:
            self.place(features, perm)

    def place(self, features, perm):
        """K7: fill this device's HBM rows (and the cold tier unless shared)."""
        if isinstance(features, FeatureMatrix):
            data = features.data
        else:
            data = features
        if not _is_torch(data):
            data = np.ascontiguousarray(data)
        p = _perm(perm)
        want = self.layout.num_rows * self.layout.bytes_per_row()
        nbytes = (data.numel() * data.element_size()) if _is_torch(data) else data.nbytes
        if nbytes != want:
            raise FormatError(f"features: data holds {nbytes} bytes, expected {want}")
        if _len(p) != self.layout.num_rows:
            raise DomainError(f"permutation length {_len(p)} != num_rows {self.layout.num_rows}")
        self._keep = [data]  # TG_COLD_INDIRECT maps the caller's matrix: keep it alive
        _check(LIB.tg_store_place(self.h, _ptr(data), _nonempty(p, np.uint64)))

    @property
    def cold_tier_bytes(self) -> int:
        """Host bytes of the cold tier in this store's format."""
        return int(LIB.tg_store_cold_tier_bytes(self.h))

    def attach_cold(self, host, fill: bool):
        """Use `host` (a SharedHostSegment or a mapped/registered array) as the
        cold tier; call with place=False at construction, before place().
        fill=True: this store writes the cold rows (one process per node);
        fill=False: another process has written them."""
        ptr, nbytes = (host.ptr, host.nbytes) if isinstance(host, SharedHostSegment) else \
            (_ptr(host), _nbytes(host))
        self._cold_ref = host
        _check(LIB.tg_store_attach_cold(self.h, C.c_void_p(ptr), nbytes, int(fill)))

    def place_file(self, path, perm):
        """K7 straight from a FEAT v1 file (io.hpp:35): rows to this device's
        HBM slots and the pinned cold tier, no N x R host copy."""
        p = _perm(perm)
        if _len(p) != self.layout.num_rows:
            raise DomainError(f"permutation length {_len(p)} != num_rows {self.layout.num_rows}")
        self._keep = [p]
        _check(LIB.tg_store_place_feat(self.h, str(path).encode(), _nonempty(p, np.uint64)))

    def place_rows(self, rows, row_of):
        """K7 from a caller's row array: new id i holds rows[row_of[i]]
        (rows: [nrows, row_bytes] host or device; row_of: N u32)."""
        R = self.layout.bytes_per_row()
        if not _is_torch(rows):
            rows = np.ascontiguousarray(rows)
        nbytes = (rows.numel() * rows.element_size()) if _is_torch(rows) else rows.nbytes
        if R == 0 or nbytes % R:
            raise FormatError(f"rows: {nbytes} bytes is not a whole number of {R}-byte rows")
        ro = np.ascontiguousarray(row_of, dtype=np.uint32) if not _is_torch(row_of) else row_of
        if _len(ro) != self.layout.num_rows:
            raise DomainError(f"row map length {_len(ro)} != num_rows {self.layout.num_rows}")
        self._keep = [rows, ro]
        _check(LIB.tg_store_place_rows(self.h, _ptr(rows), nbytes // R, _ptr(ro)))

    @property
    def local_base(self) -> int:
        return int(LIB.tg_store_local_base(self.h) or 0)

    @property
    def local_rows(self) -> int:
        return int(LIB.tg_store_local_rows(self.h))

    @property
    def cold_host_bytes(self) -> int:
        """Bytes of each cold row that cross PCIe (row_bytes, or its whole
        128 B lines when the remainder is kept in HBM)."""
        return int(LIB.tg_store_cold_host_bytes(self.h))

    def measure_cold_us(self, rows: int, reps: int = 5) -> float:
        """Mean us to read `rows` random rows of this store's cold region
        (L2 flushed per launch): the floor of a gather's cold part."""
        v = C.c_double()
        _check(LIB.tg_store_measure_cold_us(self.h, int(rows), int(reps), C.byref(v)))
        return float(v.value)

    def measure_cold_rows_us(self, rows: int, reps: int = 5) -> float:
        """The platform ceiling of the same: a plain one-warp-per-row copy of
        `rows` random rows of the cold tier (tg_store_measure_cold_rows_us)."""
        v = C.c_double()
        _check(LIB.tg_store_measure_cold_rows_us(self.h, int(rows), int(reps), C.byref(v)))
        return float(v.value)

    def set_peer(self, device_index: int, peer_local_base: int):
        _check(LIB.tg_store_set_peer(self.h, int(device_index), C.c_void_p(peer_local_base)))

    def share_cold(self, owner: "TieredFeatureStore"):
        _check(LIB.tg_store_share_cold(self.h, owner.h))
        self._cold_owner = owner

    def gather_rows(self, ids, out=None, report: TrafficReport = None):
        """K8: rows ids -> out [len(ids), row_bytes] (numpy uint8 or a CUDA tensor);
        accounting accumulated into `report` like the reference gather()."""
        idx = _u64(ids)
        n = _len(idx)
        rb = self.layout.bytes_per_row()
        if out is None:
            out = np.empty((n, rb), np.uint8)
        _check_out(out, n * rb)
        r = (report or TrafficReport())._c()
        try:
            _check(LIB.tg_gather_rows(self.h, _nonempty(idx, np.uint64), n,
                                      _nonempty(out, np.uint8), C.byref(r)))
        finally:
            if report is not None:
                report._load(r)
        return out

    def time_gather_rows(self, id_lists, out, report: TrafficReport = None,
                         flush_l2: bool = True) -> float:
        """Seconds spent in len(id_lists) synchronous tg_gather_rows calls,
        timed inside the library around each call (no Python in the timed
        region); ids are host arrays (pinned ones are read in place)."""
        lists = [np.ascontiguousarray(x, dtype=np.uint64) for x in id_lists]
        _check_out(out, max((len(x) for x in lists), default=0) * self.layout.bytes_per_row())
        ptrs = (C.c_void_p * len(lists))(*[x.ctypes.data for x in lists])
        cnts = (C.c_uint64 * len(lists))(*[len(x) for x in lists])
        r = (report or TrafficReport())._c()
        sec = C.c_double()
        try:
            _check(LIB.tg_time_gather_rows(self.h, ptrs, cnts, len(lists), _ptr(out),
                                           int(flush_l2), C.byref(r), C.byref(sec)))
        finally:
            if report is not None:
                report._load(r)
        return float(sec.value)

    def gather_rows_async(self, ids_dev, out_dev, counters_dev, err_dev):
        """Stream-ordered K8 on device tensors (no synchronisation)."""
        _check_out(out_dev, _len(ids_dev) * self.layout.bytes_per_row(), "out_dev")
        _check_out(counters_dev, 24, "counters_dev")
        _check_out(err_dev, 8, "err_dev")
        _check(LIB.tg_gather_rows_async(self.h, _ptr(ids_dev), _len(ids_dev), _ptr(out_dev),
                                        _ptr(counters_dev), _ptr(err_dev)))

    def close(self):
        if getattr(self, "h", None):
            LIB.tg_store_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ utilities
class SharedHostSegment:
    """One pinned host segment per NODE shared by all its processes
    (tg_host_shared_map: POSIX shared memory, mapped and registered in each
    process -- PAPER.md:659-663). `array` is a uint8 numpy view. The creator
    unlinks the name on close (the memory lives until every process unmaps)."""

    def __init__(self, name: str, nbytes: int, create: bool):
        p = C.c_void_p()
        _check(LIB.tg_host_shared_map(name.encode(), int(nbytes), int(create), C.byref(p)))
        self.name, self.nbytes, self.ptr, self.creator = name, int(nbytes), p.value, create
        self.array = np.frombuffer((C.c_uint8 * self.nbytes).from_address(self.ptr), np.uint8)

    def close(self):
        if self.ptr:
            self.array = None
            LIB.tg_host_shared_unmap(C.c_void_p(self.ptr), self.nbytes)
            if self.creator:
                LIB.tg_host_shared_unlink(self.name.encode())
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_alloc(nbytes: int) -> np.ndarray:
    """Pinned, mapped host buffer (cudaHostAlloc Mapped|Portable) as uint8 numpy."""
    p = C.c_void_p()
    _check(LIB.tg_host_alloc(int(nbytes), C.byref(p)))
    buf = (C.c_uint8 * int(nbytes)).from_address(p.value)
    arr = np.frombuffer(buf, dtype=np.uint8)
    arr_owner = _PinnedOwner(p.value)
    _PINNED[id(arr)] = arr_owner
    return arr


def host_register(arr: np.ndarray) -> None:
    """Pin and map caller host memory in place (cudaHostRegister,
    PAPER.md:659-668); a store placed from it then reads it as is."""
    _check(LIB.tg_host_register(C.c_void_p(arr.ctypes.data), int(arr.nbytes)))


def mapped_device_pointer(arr: np.ndarray) -> int:
    """Device address of registered/pinned host memory (0 if not mapped)."""
    return int(LIB.tg_mapped_device_ptr(C.c_void_p(arr.ctypes.data)) or 0)


def host_unregister(arr: np.ndarray) -> None:
    _check(LIB.tg_host_unregister(C.c_void_p(arr.ctypes.data)))


class _PinnedOwner:
    def __init__(self, p):
        self.p = p


_PINNED = {}


def measure_host_read_gbps(ctx: Context = None, nbytes=1 << 30, row_bytes=512, reps=5) -> float:
    c = _ctx(ctx)
    v = C.c_double()
    _check(LIB.tg_measure_host_read_gbps(c.h, int(nbytes), int(row_bytes), int(reps), C.byref(v)))
    return float(v.value)


def measure_hbm_copy_gbps(ctx: Context = None, nbytes=1 << 30, reps=5) -> float:
    c = _ctx(ctx)
    v = C.c_double()
    _check(LIB.tg_measure_hbm_copy_gbps(c.h, int(nbytes), int(reps), C.byref(v)))
    return float(v.value)
