"""TEST INFRASTRUCTURE ONLY — CPU oracles for the tiergraph hot path.

Two interchangeable checkers with one numpy-facing API:

* ``port()``  — ``_build/libtgoracle.so``, the plain-C restatement in
  ``tg_oracle.c`` (each function cites the reference file:line it follows).
* ``ref()``   — ``_ref/libtgref.so``, the UNMODIFIED reference sources from
  ``/root/reference/proj/src`` compiled out-of-tree (``Makefile``) behind the
  forwarding shim ``ref_shim.cpp``. Returns ``None`` when it was not built.

The restatement is pinned against the reference build and the reference
tests' known answers in ``tests/test_oracle.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package, and only
as the checker / CPU baseline — never as a product code path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libtgoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtgref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
vp = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
I32 = C.c_int


class OracleError(RuntimeError):
    pass


class DomainError(OracleError, ValueError):
    """Reference DomainError (types.hpp:26-29)."""


class FormatError(OracleError):
    """Reference FormatError (types.hpp:20-23)."""


class IoError(OracleError, OSError):
    """Reference IoError (types.hpp:13-16)."""


def _raise(rc: int, msg: str = ""):
    if rc == 0:
        return
    if rc == 2:
        raise DomainError(msg)
    if rc == 3:
        raise FormatError(msg)
    if rc == 4:
        raise IoError(msg)
    raise OracleError(f"rc={rc}: {msg}")


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference build when its sources exist)."""
    target = "all" if ref else "oracle"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def layout6(layout) -> np.ndarray:
    """(num_rows, local_boundary, multi_boundary, num_devices, feature_dim, elem_bytes)."""
    if hasattr(layout, "as_tuple"):
        layout = layout.as_tuple()
    return _u64(layout)


# ---------------------------------------------------------------------------
class PortOracle:
    """ctypes view of tg_oracle.c."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.L = C.CDLL(path)
        sig = {
            "tgo_mix64": (U64, [U64]),
            "tgo_derive_stream_key": (U64, [U64, u64p, U32]),
            "tgo_in_degrees": (None, [u64p, u64p, U64, u64p]),
            "tgo_transpose": (None, [u64p, u64p, U64, u64p, u64p]),
            "tgo_from_edge_list": (I32, [U64, u64p, u64p, U64, u64p, C.POINTER(vp), C.POINTER(U64)]),
            "tgo_make_test_features": (None, [U64, U64, vp]),
            "tgo_draw_random_train_ids": (I32, [U64, U64, U64, u64p]),
            "tgo_reverse_pagerank": (I32, [u64p, u64p, U64, vp, U64, U32, C.c_double, f64p]),
            "tgo_degree_score": (None, [u64p, U64, f64p]),
            "tgo_score_ordering": (I32, [f64p, U64, u64p]),
            "tgo_validate_permutation": (I32, [u64p, U64]),
            "tgo_permutation_from_scores": (I32, [f64p, U64, u64p]),
            "tgo_invert": (I32, [u64p, U64, u64p]),
            "tgo_reorder_graph": (I32, [u64p, u64p, U64, u64p, u64p, u64p]),
            "tgo_reorder_features": (I32, [vp, U64, U64, u64p, vp]),
            "tgo_validate_layout": (I32, [u64p]),
            "tgo_resolve": (I32, [u64p, U64, U32, u64p]),
            "tgo_plan_layout": (I32, [U64, C.c_double, C.c_double, U32, U64, U32, U64, u64p]),
            "tgo_gather": (I32, [u64p, u64p, U64, U32, u64p]),
            "tgo_simulate_trace": (I32, [u64p, U64, u64p, u64p]),
            "tgo_counts_in_row_order": (I32, [u64p, U64, u64p, U64, u64p]),
            "tgo_hot_fraction_sweep": (I32, [u64p, U64, u64p, f64p, U64, C.c_double, U32, U64, U32,
                                             U64, u64p, u64p, f64p]),
            "tgo_build_minibatch": (I32, [u64p, u64p, U64, u64p, U64, u32p, U32, U64, U64, U64,
                                          C.POINTER(vp), C.POINTER(U64)]),
            "tgo_sample_index_subset": (U64, [C.POINTER(U64), U64, U64, u64p]),
            "tgo_shuffle": (None, [C.POINTER(U64), u64p, U64]),
            "tgo_build_minibatch_tier_reads": (I32, [u64p, u64p, U64, u64p, U64, u32p, U32, U64, U64,
                                                      U64, u64p, U32, u64p]),
            "tgo_free": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    # -- rng / fixtures
    def mix64(self, x):
        return self.L.tgo_mix64(int(x))

    def derive_stream_key(self, seed, coords):
        c = _u64(list(coords) or [0])
        return self.L.tgo_derive_stream_key(int(seed), c, len(coords))

    def sample_index_subset(self, key, population, k):
        st = U64(key)
        out = np.zeros(max(1, min(k, population)), np.uint64)
        n = self.L.tgo_sample_index_subset(C.byref(st), population, k, out)
        return out[:n]

    def shuffle(self, key, items):
        st = U64(key)
        a = _u64(items).copy()
        self.L.tgo_shuffle(C.byref(st), a, len(a))
        return a

    def make_test_features(self, rows, dim):
        out = np.empty((rows, dim), np.float32)
        self.L.tgo_make_test_features(rows, dim, out.ctypes.data)
        return out

    def draw_random_train_ids(self, n, count, seed):
        out = np.empty(max(count, 1), np.uint64)
        _raise(self.L.tgo_draw_random_train_ids(n, count, seed, out), "draw_random_train_ids")
        return out[:count]

    # -- graph core
    def from_edge_list(self, n, src, dst):
        src, dst = _u64(src), _u64(dst)
        off = np.empty(n + 1, np.uint64)
        p, e = vp(), U64()
        _raise(self.L.tgo_from_edge_list(n, src, dst, len(src), off, C.byref(p), C.byref(e)),
               "edge out of range")
        tgt = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), shape=(max(e.value, 1),))
        tgt = tgt[: e.value].copy()
        self.L.tgo_free(p)
        return off, tgt

    def transpose(self, off, tgt):
        off, tgt = _u64(off), _u64(tgt)
        n = len(off) - 1
        t_off = np.empty(n + 1, np.uint64)
        t_tgt = np.empty(max(len(tgt), 1), np.uint64)
        self.L.tgo_transpose(off, tgt if len(tgt) else np.zeros(1, np.uint64), n, t_off, t_tgt)
        return t_off, t_tgt[: len(tgt)]

    def in_degrees(self, off, tgt):
        off, tgt = _u64(off), _u64(tgt)
        n = len(off) - 1
        out = np.empty(max(n, 1), np.uint64)
        self.L.tgo_in_degrees(off, tgt if len(tgt) else np.zeros(1, np.uint64), n, out)
        return out[:n]

    # -- scoring
    def reverse_pagerank(self, off, tgt, iterations=5, damp=0.85):
        return self._rpr(off, tgt, None, iterations, damp)

    def weighted_reverse_pagerank(self, off, tgt, tid, iterations=5, damp=0.85):
        return self._rpr(off, tgt, _u64(tid), iterations, damp)

    def _rpr(self, off, tgt, tid, iterations, damp):
        off, tgt = _u64(off), _u64(tgt)
        n = len(off) - 1
        out = np.empty(max(n, 1), np.float64)
        tp = tid.ctypes.data if tid is not None and len(tid) else (1 if tid is not None else None)
        nt = len(tid) if tid is not None else 0
        rc = self.L.tgo_reverse_pagerank(off, tgt if len(tgt) else np.zeros(1, np.uint64), n,
                                         tp, nt, iterations, damp, out)
        _raise(rc, "pagerank")
        return out[:n]

    def degree_score(self, off):
        off = _u64(off)
        out = np.empty(max(len(off) - 1, 1), np.float64)
        self.L.tgo_degree_score(off, len(off) - 1, out)
        return out[: len(off) - 1]

    def score_ordering(self, scores):
        s = _f64(scores)
        out = np.empty(max(len(s), 1), np.uint64)
        _raise(self.L.tgo_score_ordering(s if len(s) else np.zeros(1), len(s), out), "score")
        return out[: len(s)]

    # -- reorder
    def permutation_from_scores(self, scores):
        s = _f64(scores)
        out = np.empty(max(len(s), 1), np.uint64)
        _raise(self.L.tgo_permutation_from_scores(s if len(s) else np.zeros(1), len(s), out), "score")
        return out[: len(s)]

    def validate_permutation(self, perm):
        p = _u64(perm)
        _raise(self.L.tgo_validate_permutation(p if len(p) else np.zeros(1, np.uint64), len(p)),
               "permutation")

    def invert(self, perm):
        p = _u64(perm)
        out = np.empty(max(len(p), 1), np.uint64)
        _raise(self.L.tgo_invert(p if len(p) else np.zeros(1, np.uint64), len(p), out), "perm")
        return out[: len(p)]

    def reorder_graph(self, off, tgt, perm):
        off, tgt, p = _u64(off), _u64(tgt), _u64(perm)
        n = len(off) - 1
        if len(p) != n:
            raise DomainError("permutation length != num_nodes")
        o = np.empty(n + 1, np.uint64)
        t = np.empty(max(len(tgt), 1), np.uint64)
        _raise(self.L.tgo_reorder_graph(off, tgt if len(tgt) else np.zeros(1, np.uint64), n,
                                        p if n else np.zeros(1, np.uint64), o, t), "perm")
        return o, t[: len(tgt)]

    def reorder_features(self, data, perm):
        data = np.ascontiguousarray(data)
        p = _u64(perm)
        rows = data.shape[0]
        if len(p) != rows:
            raise DomainError("permutation length != num_rows")
        rb = data.nbytes // max(rows, 1)
        out = np.empty_like(data)
        _raise(self.L.tgo_reorder_features(data.ctypes.data, rows, rb,
                                           p if rows else np.zeros(1, np.uint64), out.ctypes.data),
               "perm")
        return out

    # -- tiering
    def validate_layout(self, layout):
        _raise(self.L.tgo_validate_layout(layout6(layout)), "layout")

    def resolve(self, layout, row, dev):
        out = np.zeros(3, np.uint64)
        _raise(self.L.tgo_resolve(layout6(layout), row, dev, out), "resolve")
        return tuple(int(x) for x in out)

    def plan_layout(self, num_rows, hot, rep, devices, dim, elem_bytes, budget=0):
        out = np.zeros(6, np.uint64)
        _raise(self.L.tgo_plan_layout(num_rows, hot, rep, devices, dim, elem_bytes, budget, out),
               "plan_layout")
        return tuple(int(x) for x in out)

    def gather(self, layout, ids, dev, report=None):
        r = _u64(report if report is not None else np.zeros(6)).copy()
        ids = _u64(ids)
        rc = self.L.tgo_gather(layout6(layout), ids if len(ids) else np.zeros(1, np.uint64),
                               len(ids), dev, r)
        _raise(rc, "gather")
        return r

    def simulate_trace(self, counts, layout):
        c = _u64(counts)
        r = np.zeros(6, np.uint64)
        _raise(self.L.tgo_simulate_trace(c if len(c) else np.zeros(1, np.uint64), len(c),
                                         layout6(layout), r), "simulate_trace")
        return r

    def counts_in_row_order(self, counts, ordering):
        c, o = _u64(counts), _u64(ordering)
        out = np.empty(max(len(o), 1), np.uint64)
        _raise(self.L.tgo_counts_in_row_order(c, len(c), o, len(o), out), "counts")
        return out[: len(o)]

    def hot_fraction_sweep(self, counts, ordering, fractions, replicated, devices, dim,
                           elem_bytes, budget=0):
        c, o, f = _u64(counts), _u64(ordering), _f64(fractions)
        nf = len(f)
        lay = np.zeros(6 * max(nf, 1), np.uint64)
        rep = np.zeros(6 * max(nf, 1), np.uint64)
        rf = np.zeros(max(nf, 1), np.float64)
        _raise(self.L.tgo_hot_fraction_sweep(c, len(c), o, f if nf else np.zeros(1), nf,
                                             replicated, devices, dim, elem_bytes, budget,
                                             lay, rep, rf), "sweep")
        return lay[: 6 * nf].reshape(nf, 6), rep[: 6 * nf].reshape(nf, 6), rf[:nf]

    # -- sampling
    def build_minibatch(self, gt_off, gt_tgt, seeds, fanouts, rng_seed=0, epoch=0, batch=0):
        go, gt, s = _u64(gt_off), _u64(gt_tgt), _u64(seeds)
        f = np.ascontiguousarray(np.asarray(fanouts, np.uint32))
        p, m = vp(), U64()
        rc = self.L.tgo_build_minibatch(go, gt if len(gt) else np.zeros(1, np.uint64), len(go) - 1,
                                        s if len(s) else np.zeros(1, np.uint64), len(s),
                                        f if len(f) else np.zeros(1, np.uint32), len(f),
                                        rng_seed, epoch, batch, C.byref(p), C.byref(m))
        _raise(rc, "build_minibatch")
        out = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), shape=(max(m.value, 1),))
        out = out[: m.value].copy()
        self.L.tgo_free(p)
        return out

    def structure_tier_reads(self, gt_off, gt_tgt, seeds, fanouts, layout, device,
                             rng_seed=0, epoch=0, batch=0):
        """Neighbour ids build_minibatch reads per tier {local, peer, host}
        when gt's rows are placed by `layout` (lb, mb, D) for `device`
        (graph-structure tiering)."""
        go, gt, s = _u64(gt_off), _u64(gt_tgt), _u64(seeds)
        f = np.ascontiguousarray(np.asarray(fanouts, np.uint32))
        lay = layout6(layout)
        lay3 = np.array([lay[1], lay[2], lay[3]], np.uint64)
        reads = np.zeros(3, np.uint64)
        rc = self.L.tgo_build_minibatch_tier_reads(
            go, gt if len(gt) else np.zeros(1, np.uint64), len(go) - 1,
            s if len(s) else np.zeros(1, np.uint64), len(s), f if len(f) else np.zeros(1, np.uint32),
            len(f), rng_seed, epoch, batch, lay3, int(device), reads)
        _raise(rc, "build_minibatch")
        return reads

    def epoch_minibatches(self, gt_off, gt_tgt, tid, fanouts, batch_size, rng_seed, epoch,
                          max_batches=0):
        """run_training_trace's per-epoch schedule (sampling.cpp:106-123)."""
        key = self.derive_stream_key(rng_seed, [0x5348, epoch])
        order = self.shuffle(key, tid)
        nb = (len(order) + batch_size - 1) // batch_size
        if max_batches:
            nb = min(nb, max_batches)
        return [self.build_minibatch(gt_off, gt_tgt, order[b * batch_size:(b + 1) * batch_size],
                                     fanouts, rng_seed, epoch, b) for b in range(nb)]


# ---------------------------------------------------------------------------
class RefOracle:
    """ctypes view of the reference library build (ref_shim.cpp)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        L = self.L = C.CDLL(path)
        sig = {
            "tgref_last_error": (C.c_char_p, []),
            "tgref_free": (None, [vp]),
            "tgref_set_worker_count": (None, [I32]),
            "tgref_worker_count": (I32, []),
            "tgref_graph_create": (vp, [u64p, vp, U64, U64]),
            "tgref_graph_destroy": (None, [vp]),
            "tgref_graph_num_edges": (U64, [vp]),
            "tgref_graph_num_nodes": (U64, [vp]),
            "tgref_graph_export": (None, [vp, u64p, vp]),
            "tgref_from_edge_list": (I32, [U64, u64p, u64p, U64, C.POINTER(vp)]),
            "tgref_generate_power_law": (I32, [U64, U64, U64, C.POINTER(vp)]),
            "tgref_graph_transpose": (vp, [vp]),
            "tgref_validate_csr": (I32, [vp, I32]),
            "tgref_in_degrees": (None, [vp, u64p]),
            "tgref_train_ids_from": (I32, [u64p, U64, U64, C.POINTER(vp), C.POINTER(U64)]),
            "tgref_draw_random_train_ids": (I32, [U64, U64, U64, u64p]),
            "tgref_degree_score": (None, [vp, f64p]),
            "tgref_reverse_pagerank": (I32, [vp, U32, C.c_double, f64p]),
            "tgref_weighted_reverse_pagerank": (I32, [vp, U32, C.c_double, vp, U64, f64p]),
            "tgref_score_ordering": (I32, [f64p, U64, u64p]),
            "tgref_permutation_from_scores": (I32, [f64p, U64, u64p]),
            "tgref_validate_permutation": (I32, [u64p, U64]),
            "tgref_invert": (I32, [u64p, U64, u64p]),
            "tgref_reorder_graph": (I32, [vp, u64p, U64, C.POINTER(vp)]),
            "tgref_sequential_reorder_oracle": (I32, [vp, u64p, U64, C.POINTER(vp)]),
            "tgref_features_create": (vp, [vp, U64, U64, U32]),
            "tgref_make_test_features": (vp, [U64, U64]),
            "tgref_features_destroy": (None, [vp]),
            "tgref_features_data": (vp, [vp]),
            "tgref_features_nbytes": (U64, [vp]),
            "tgref_reorder_features": (I32, [vp, u64p, U64, C.POINTER(vp)]),
            "tgref_features_gather": (I32, [vp, u64p, vp, U64, U32, vp, u64p]),
            "tgref_features_gather_inv": (I32, [vp, U64, U64, vp, u64p, vp, U64, U32, vp, u64p]),
            "tgref_validate_layout": (I32, [u64p]),
            "tgref_validate_cost_model": (I32, [C.c_double, C.c_double, C.c_double]),
            "tgref_resolve": (I32, [u64p, U64, U32, u64p]),
            "tgref_plan_layout": (I32, [U64, C.c_double, C.c_double, U32, U64, U32, U64, u64p]),
            "tgref_gather": (I32, [u64p, vp, U64, U32, u64p]),
            "tgref_simulate_trace": (I32, [u64p, U64, u64p, u64p]),
            "tgref_counts_in_row_order": (I32, [u64p, U64, u64p, U64, u64p]),
            "tgref_hot_fraction_sweep": (I32, [u64p, U64, u64p, f64p, U64, C.c_double, U32, U64,
                                               U32, U64, u64p, u64p, f64p]),
            "tgref_hit_ratio": (C.c_double, [u64p]),
            "tgref_est_transfer_seconds": (C.c_double, [u64p, C.c_double, C.c_double, C.c_double]),
            "tgref_build_minibatch": (I32, [vp, u64p, U64, u32p, U32, U64, U64, U64,
                                            C.POINTER(vp), C.POINTER(U64)]),
            "tgref_epoch_minibatches": (I32, [vp, u64p, U64, u32p, U32, U64, U64, U64, U64,
                                              C.POINTER(vp), C.POINTER(U64), C.POINTER(vp)]),
            "tgref_run_training_trace": (I32, [vp, u64p, U64, u32p, U32, U64, U64, U64, I32, u64p]),
            "tgref_mix64": (U64, [U64]),
            "tgref_save_csr": (I32, [vp, C.c_char_p]),
            "tgref_load_csr": (I32, [C.c_char_p, C.POINTER(vp)]),
            "tgref_save_features": (I32, [vp, C.c_char_p]),
            "tgref_load_features": (I32, [C.c_char_p, C.POINTER(vp)]),
            "tgref_save_perm": (I32, [u64p, U64, C.c_char_p]),
            "tgref_derive_stream_key": (U64, [U64, u64p, U32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    def _chk(self, rc):
        if rc:
            _raise(rc, self.L.tgref_last_error().decode())

    def _take(self, p, n):
        if n == 0:
            self.L.tgref_free(p)
            return np.zeros(0, np.uint64)
        a = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), shape=(n,)).copy()
        self.L.tgref_free(p)
        return a

    def set_worker_count(self, n):
        self.L.tgref_set_worker_count(int(n))

    # io.cpp containers ----------------------------------------------------
    def save_csr(self, off, tgt, path):
        g = self.graph(off, tgt)
        self._chk(self.L.tgref_save_csr(g.h, str(path).encode()))

    def load_csr(self, path):
        """(offsets, targets) read by the reference; raises its error."""
        h = C.c_void_p()
        self._chk(self.L.tgref_load_csr(str(path).encode(), C.byref(h)))
        return self._export(_RefGraph(self, h.value).h)

    def save_features(self, data, rows, dim, elem_bytes, path):
        data = np.ascontiguousarray(data).reshape(-1).view(np.uint8)
        h = self.L.tgref_features_create(data.ctypes.data, rows, dim, elem_bytes)
        try:
            self._chk(self.L.tgref_save_features(h, str(path).encode()))
        finally:
            self.L.tgref_features_destroy(h)

    def load_features_error(self, path):
        """The reference's load_features() outcome: None or (code, message)."""
        h = C.c_void_p()
        rc = self.L.tgref_load_features(str(path).encode(), C.byref(h))
        if rc:
            return rc, self.L.tgref_last_error().decode()
        self.L.tgref_features_destroy(h)
        return None

    def save_perm(self, perm, path):
        p = _u64(perm)
        self._chk(self.L.tgref_save_perm(p, len(p), str(path).encode()))

    # graph handles -------------------------------------------------------
    def graph(self, off, tgt):
        off, tgt = _u64(off), _u64(tgt)
        return _RefGraph(self, self.L.tgref_graph_create(off, tgt.ctypes.data if len(tgt) else None,
                                                         len(off) - 1, len(tgt)))

    def _export(self, h):
        n, e = self.L.tgref_graph_num_nodes(h), self.L.tgref_graph_num_edges(h)
        off = np.empty(n + 1, np.uint64)
        tgt = np.empty(max(e, 1), np.uint64)
        self.L.tgref_graph_export(h, off, tgt.ctypes.data)
        self.L.tgref_graph_destroy(h)
        return off, tgt[:e]

    def mix64(self, x):
        return self.L.tgref_mix64(int(x))

    def derive_stream_key(self, seed, coords):
        c = _u64(list(coords) or [0])
        return self.L.tgref_derive_stream_key(int(seed), c, len(coords))

    def from_edge_list(self, n, src, dst):
        h = vp()
        self._chk(self.L.tgref_from_edge_list(n, _u64(src), _u64(dst), len(src), C.byref(h)))
        return self._export(h)

    def generate_power_law(self, n, m, seed):
        h = vp()
        self._chk(self.L.tgref_generate_power_law(n, m, seed, C.byref(h)))
        return self._export(h)

    def transpose(self, off, tgt):
        g = self.graph(off, tgt)
        return self._export(self.L.tgref_graph_transpose(g.h))

    def in_degrees(self, off, tgt):
        g = self.graph(off, tgt)
        out = np.empty(max(len(off) - 1, 1), np.uint64)
        self.L.tgref_in_degrees(g.h, out)
        return out[: len(off) - 1]

    def make_test_features(self, rows, dim):
        h = self.L.tgref_make_test_features(rows, dim)
        nb = self.L.tgref_features_nbytes(h)
        a = np.ctypeslib.as_array(C.cast(self.L.tgref_features_data(h), C.POINTER(C.c_uint8)),
                                  shape=(nb,)).copy()
        self.L.tgref_features_destroy(h)
        return a.view(np.float32).reshape(rows, dim)

    def draw_random_train_ids(self, n, count, seed):
        out = np.empty(max(count, 1), np.uint64)
        self._chk(self.L.tgref_draw_random_train_ids(n, count, seed, out))
        return out[:count]

    def train_ids_from(self, raw, num_nodes):
        p, m = vp(), U64()
        self._chk(self.L.tgref_train_ids_from(_u64(raw), len(raw), num_nodes, C.byref(p), C.byref(m)))
        return self._take(p, m.value)

    def reverse_pagerank(self, off, tgt, iterations=5, damp=0.85):
        g = self.graph(off, tgt)
        out = np.empty(max(len(off) - 1, 1), np.float64)
        self._chk(self.L.tgref_reverse_pagerank(g.h, iterations, damp, out))
        return out[: len(off) - 1]

    def weighted_reverse_pagerank(self, off, tgt, tid, iterations=5, damp=0.85):
        g = self.graph(off, tgt)
        return g.weighted_reverse_pagerank(tid, iterations, damp)

    def degree_score(self, off):
        off = _u64(off)
        g = self.graph(off, np.zeros(int(off[-1]), np.uint64))
        out = np.empty(max(len(off) - 1, 1), np.float64)
        self.L.tgref_degree_score(g.h, out)
        return out[: len(off) - 1]

    def score_ordering(self, scores):
        s = _f64(scores)
        out = np.empty(max(len(s), 1), np.uint64)
        self._chk(self.L.tgref_score_ordering(s if len(s) else np.zeros(1), len(s), out))
        return out[: len(s)]

    def permutation_from_scores(self, scores):
        s = _f64(scores)
        out = np.empty(max(len(s), 1), np.uint64)
        self._chk(self.L.tgref_permutation_from_scores(s if len(s) else np.zeros(1), len(s), out))
        return out[: len(s)]

    def validate_permutation(self, perm):
        p = _u64(perm)
        self._chk(self.L.tgref_validate_permutation(p if len(p) else np.zeros(1, np.uint64), len(p)))

    def invert(self, perm):
        p = _u64(perm)
        out = np.empty(max(len(p), 1), np.uint64)
        self._chk(self.L.tgref_invert(p if len(p) else np.zeros(1, np.uint64), len(p), out))
        return out[: len(p)]

    def reorder_graph(self, off, tgt, perm):
        g = self.graph(off, tgt)
        h = vp()
        p = _u64(perm)
        self._chk(self.L.tgref_reorder_graph(g.h, p if len(p) else np.zeros(1, np.uint64), len(p),
                                             C.byref(h)))
        return self._export(h)

    def reorder_features(self, data, perm):
        data = np.ascontiguousarray(data)
        rows = data.shape[0]
        rb = data.nbytes // max(rows, 1)
        h = self.L.tgref_features_create(data.ctypes.data, rows, rb, 1)
        try:
            out = vp()
            p = _u64(perm)
            self._chk(self.L.tgref_reorder_features(h, p if len(p) else np.zeros(1, np.uint64),
                                                    len(p), C.byref(out)))
            nb = self.L.tgref_features_nbytes(out)
            a = np.ctypeslib.as_array(C.cast(self.L.tgref_features_data(out), C.POINTER(C.c_uint8)),
                                      shape=(max(nb, 1),))[:nb].copy()
            self.L.tgref_features_destroy(out)
            return a.view(data.dtype).reshape(data.shape)
        finally:
            self.L.tgref_features_destroy(h)

    def validate_layout(self, layout):
        self._chk(self.L.tgref_validate_layout(layout6(layout)))

    def resolve(self, layout, row, dev):
        out = np.zeros(3, np.uint64)
        self._chk(self.L.tgref_resolve(layout6(layout), row, dev, out))
        return tuple(int(x) for x in out)

    def plan_layout(self, num_rows, hot, rep, devices, dim, elem_bytes, budget=0):
        out = np.zeros(6, np.uint64)
        self._chk(self.L.tgref_plan_layout(num_rows, hot, rep, devices, dim, elem_bytes, budget, out))
        return tuple(int(x) for x in out)

    def gather(self, layout, ids, dev, report=None):
        r = _u64(report if report is not None else np.zeros(6)).copy()
        ids = _u64(ids)
        self._chk(self.L.tgref_gather(layout6(layout), ids.ctypes.data if len(ids) else None,
                                      len(ids), dev, r))
        return r

    def simulate_trace(self, counts, layout):
        c = _u64(counts)
        r = np.zeros(6, np.uint64)
        self._chk(self.L.tgref_simulate_trace(c if len(c) else np.zeros(1, np.uint64), len(c),
                                              layout6(layout), r))
        return r

    def counts_in_row_order(self, counts, ordering):
        c, o = _u64(counts), _u64(ordering)
        out = np.empty(max(len(o), 1), np.uint64)
        self._chk(self.L.tgref_counts_in_row_order(c, len(c), o, len(o), out))
        return out[: len(o)]

    def hot_fraction_sweep(self, counts, ordering, fractions, replicated, devices, dim,
                           elem_bytes, budget=0):
        c, o, f = _u64(counts), _u64(ordering), _f64(fractions)
        nf = len(f)
        lay = np.zeros(6 * max(nf, 1), np.uint64)
        rep = np.zeros(6 * max(nf, 1), np.uint64)
        rf = np.zeros(max(nf, 1), np.float64)
        self._chk(self.L.tgref_hot_fraction_sweep(c, len(c), o, f if nf else np.zeros(1), nf,
                                                  replicated, devices, dim, elem_bytes, budget,
                                                  lay, rep, rf))
        return lay[: 6 * nf].reshape(nf, 6), rep[: 6 * nf].reshape(nf, 6), rf[:nf]

    def hit_ratio(self, report):
        return self.L.tgref_hit_ratio(_u64(report))

    def est_transfer_seconds(self, report, local=900.0, peer=150.0, host=16.0):
        return self.L.tgref_est_transfer_seconds(_u64(report), local, peer, host)

    def build_minibatch(self, gt_off, gt_tgt, seeds, fanouts, rng_seed=0, epoch=0, batch=0):
        g = self.graph(gt_off, gt_tgt)
        return g.build_minibatch(seeds, fanouts, rng_seed, epoch, batch)

    def epoch_minibatches(self, gt_off, gt_tgt, tid, fanouts, batch_size, rng_seed, epoch,
                          max_batches=0):
        g = self.graph(gt_off, gt_tgt)
        return g.epoch_minibatches(tid, fanouts, batch_size, rng_seed, epoch, max_batches)

    def run_training_trace(self, off, tgt, tid, fanouts, batch_size, epochs, rng_seed, dedup=True):
        g = self.graph(off, tgt)
        f = np.ascontiguousarray(np.asarray(fanouts, np.uint32))
        out = np.zeros(len(off) - 1, np.uint64)
        self._chk(self.L.tgref_run_training_trace(g.h, _u64(tid), len(tid), f, len(f), batch_size,
                                                  epochs, rng_seed, int(dedup), out))
        return out


class _RefGraph:
    """A reference CsrGraph held across calls (construction is not timed)."""

    def __init__(self, lib: RefOracle, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.L.tgref_graph_destroy(self.h)
        except Exception:
            pass

    def weighted_reverse_pagerank(self, tid, iterations=5, damp=0.85, out=None):
        t = _u64(tid)
        n = self.lib.L.tgref_graph_num_nodes(self.h)
        out = np.empty(max(n, 1), np.float64) if out is None else out
        self.lib._chk(self.lib.L.tgref_weighted_reverse_pagerank(
            self.h, iterations, damp, t.ctypes.data if len(t) else None, len(t), out))
        return out[:n]

    def build_minibatch(self, seeds, fanouts, rng_seed=0, epoch=0, batch=0):
        s = _u64(seeds)
        f = np.ascontiguousarray(np.asarray(fanouts, np.uint32))
        p, m = vp(), U64()
        self.lib._chk(self.lib.L.tgref_build_minibatch(
            self.h, s if len(s) else np.zeros(1, np.uint64), len(s),
            f if len(f) else np.zeros(1, np.uint32), len(f), rng_seed, epoch, batch,
            C.byref(p), C.byref(m)))
        return self.lib._take(p, m.value)

    def epoch_minibatches(self, tid, fanouts, batch_size, rng_seed, epoch, max_batches=0):
        t = _u64(tid)
        f = np.ascontiguousarray(np.asarray(fanouts, np.uint32))
        po, nb, pi = vp(), U64(), vp()
        self.lib._chk(self.lib.L.tgref_epoch_minibatches(
            self.h, t, len(t), f, len(f), batch_size, rng_seed, epoch, max_batches,
            C.byref(po), C.byref(nb), C.byref(pi)))
        off = self.lib._take(po, nb.value + 1)
        ids = self.lib._take(pi, int(off[-1]))
        return [ids[off[b]:off[b + 1]] for b in range(nb.value)]


class RefFeatures:
    """A reference FeatureMatrix held across calls (for the CPU gather baseline)."""

    def __init__(self, lib: RefOracle, data: np.ndarray):
        data = np.ascontiguousarray(data)
        self.lib = lib
        self.rows = data.shape[0]
        self.row_bytes = data.nbytes // max(self.rows, 1)
        self.h = lib.L.tgref_features_create(data.ctypes.data, self.rows, self.row_bytes, 1)

    def reordered(self, perm) -> "RefFeatures":
        out = vp()
        p = _u64(perm)
        self.lib._chk(self.lib.L.tgref_reorder_features(self.h, p, len(p), C.byref(out)))
        r = RefFeatures.__new__(RefFeatures)
        r.lib, r.rows, r.row_bytes, r.h = self.lib, self.rows, self.row_bytes, out.value
        return r

    def gather(self, layout, ids: np.ndarray, dev: int, out: np.ndarray, report: np.ndarray):
        self.lib._chk(self.lib.L.tgref_features_gather(self.h, layout6(layout), ids.ctypes.data,
                                                       len(ids), dev, out.ctypes.data, report))

    def __del__(self):
        try:
            self.lib.L.tgref_features_destroy(self.h)
        except Exception:
            pass


class RefFeaturesInv:
    """The CPU byte gather over the caller's ORIGINAL matrix (no copy):
    new row id = old row inv[id], byte-identical to RefFeatures.reordered(perm)
    (reorder.cpp:113-115) without a second N x R matrix in host RAM."""

    def __init__(self, lib: RefOracle, data: np.ndarray, row_of):
        """row_of[id] = the row of `data` holding new row id (the inverse
        permutation for an original matrix)."""
        self.lib = lib
        self.data = data  # caller-owned, kept alive; rows x row_bytes (any dtype)
        self.rows = data.shape[0]
        self.row_bytes = data.nbytes // max(self.rows, 1)
        self.inv = _u64(row_of)

    def gather(self, layout, ids: np.ndarray, dev: int, out: np.ndarray, report: np.ndarray):
        ids = _u64(ids)
        if len(ids) and int(ids.max()) >= len(self.inv):
            raise DomainError(f"row {int(ids.max())} out of range")
        self.lib._chk(self.lib.L.tgref_features_gather_inv(
            self.data.ctypes.data, self.rows, self.row_bytes, self.inv.ctypes.data,
            layout6(layout), ids.ctypes.data, len(ids), dev, out.ctypes.data, report))


_port = None
_ref = None


def port() -> PortOracle:
    global _port
    if _port is None:
        _port = PortOracle()
    return _port


def ref() -> RefOracle | None:
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = RefOracle()
    return _ref
