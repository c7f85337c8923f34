"""Synthetic inputs of the named shapes (fixtures, not the hot path).

* ``rmat_graph`` — Graph500-style R-MAT (a,b,c,d = .57,.19,.19,.05) with a
  counter-based splitmix64 stream per (edge, level), so the same seed gives
  the same graph on CPU and GPU. Draws with an endpoint >= N are rejected;
  the CSR is canonicalised like the reference's from_edge_list
  (csr_graph.cpp:36-65: rows sorted ascending, duplicates dropped, self-loops
  kept). E is therefore counted AFTER rejection and de-duplication.
* ``test_features`` — the reference's closed-form f32 fill
  (feature_matrix.cpp:16-28): value(r, c) = float(mix64(r) >> 40) + c.

Generation uses torch tensors (GPU when present) purely as array plumbing.
"""
from __future__ import annotations

import numpy as np

_M30 = (1 << 34) - 1
_M27 = (1 << 37) - 1
_M31 = (1 << 33) - 1


def _i64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= 1 << 63 else x


_C0 = _i64(0x9E3779B97F4A7C15)
_C1 = _i64(0xBF58476D1CE4E5B9)
_C2 = _i64(0x94D049BB133111EB)


def mix64_torch(x):
    """splitmix64 finalizer (rng.hpp:13-18) on int64 tensors (wrapping arithmetic)."""
    x = x + _C0
    x = (x ^ ((x >> 30) & _M30)) * _C1
    x = (x ^ ((x >> 27) & _M27)) * _C2
    return x ^ ((x >> 31) & _M31)


def mix64_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def rmat_graph(num_nodes: int, num_draws: int, seed: int = 1, a=0.57, b=0.19, c=0.19,
               device=None, chunk: int = 1 << 25):
    """Returns (offsets u64 [N+1], targets u64 [E]) as numpy arrays."""
    import torch
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    scale = max(1, int(np.ceil(np.log2(max(num_nodes, 2)))))
    ab, abc = a + b, a + b + c
    keys = []
    key_seed = int(mix64_np(np.array([seed ^ 0x524D4154], np.uint64))[0])
    for start in range(0, num_draws, chunk):
        cnt = min(chunk, num_draws - start)
        idx = torch.arange(start, start + cnt, device=device, dtype=torch.int64)
        src = torch.zeros(cnt, device=device, dtype=torch.int64)
        dst = torch.zeros(cnt, device=device, dtype=torch.int64)
        base = mix64_torch(idx * scale + _i64(key_seed))
        for lvl in range(scale):
            r = mix64_torch(base + lvl)
            u = ((r >> 11) & ((1 << 53) - 1)).to(torch.float64) * (2.0 ** -53)
            sbit = (u >= ab).to(torch.int64)
            dbit = (((u >= a) & (u < ab)) | (u >= abc)).to(torch.int64)
            src = (src << 1) | sbit
            dst = (dst << 1) | dbit
        ok = (src < num_nodes) & (dst < num_nodes)
        keys.append(src[ok] * num_nodes + dst[ok])
    key = torch.unique(torch.cat(keys))  # sorted ascending: rows sorted, dedup
    src = key // num_nodes
    dst = key - src * num_nodes
    deg = torch.bincount(src, minlength=num_nodes)
    off = torch.zeros(num_nodes + 1, dtype=torch.int64, device=device)
    off[1:] = torch.cumsum(deg, 0)
    return (off.cpu().numpy().astype(np.uint64), dst.cpu().numpy().astype(np.uint64))


def test_features(num_rows: int, dim: int, out: np.ndarray = None, rows_per_chunk=1 << 20):
    """feature_matrix.cpp:16-28 closed form, f32 [num_rows, dim] (optionally into `out`)."""
    if out is None:
        out = np.empty((num_rows, dim), np.float32)
    else:
        out = out.reshape(-1).view(np.float32).reshape(num_rows, dim)
    cols = np.arange(dim, dtype=np.float32)
    for r0 in range(0, num_rows, rows_per_chunk):
        r1 = min(num_rows, r0 + rows_per_chunk)
        base = (mix64_np(np.arange(r0, r1, dtype=np.uint64)) >> np.uint64(40)).astype(np.float32)
        np.add(base[:, None], cols[None, :], out=out[r0:r1])
    return out


def expected_rows(old_ids: np.ndarray, dim: int) -> np.ndarray:
    """Closed-form rows for old ids (to verify gathers without a second copy)."""
    base = (mix64_np(np.asarray(old_ids, np.uint64)) >> np.uint64(40)).astype(np.float32)
    return base[:, None] + np.arange(dim, dtype=np.float32)[None, :]


def test_features_pinned_gpu(num_rows: int, dim: int, out: np.ndarray, device="cuda",
                             rows_per_chunk=1 << 21):
    """The same closed-form f32 fill as test_features, computed on the GPU and
    copied chunk by chunk into `out` (a pinned host buffer of num_rows*dim*4
    bytes) — for the papers100M-shaped matrix (57 GB) a numpy fill is minutes."""
    import torch
    dst = torch.from_numpy(out.reshape(-1).view(np.float32)).view(num_rows, dim)
    cols = torch.arange(dim, dtype=torch.float32, device=device)
    for r0 in range(0, num_rows, rows_per_chunk):
        r1 = min(num_rows, r0 + rows_per_chunk)
        r = torch.arange(r0, r1, dtype=torch.int64, device=device)
        base = ((mix64_torch(r) >> 40) & ((1 << 24) - 1)).to(torch.float32)
        dst[r0:r1].copy_(base[:, None] + cols[None, :])
    torch.cuda.synchronize()
    return out


# ---------------------------------------------------------------- C4 (fp16)
# MAG240M-shaped features: 768-d fp16. The reference's FeatureMatrix is
# byte-opaque (elem_bytes, feature_matrix.hpp:13-20) and its maker is f32
# only (feature_matrix.cpp:16-28), so the fp16 fixture is the same closed form
# narrowed to values fp16 holds exactly: base = mix64(r) >> 54 (0..1023),
# value = base + c (c < 768, so every value is an integer <= 1790).
def expected_rows_f16(old_ids: np.ndarray, dim: int) -> np.ndarray:
    base = (mix64_np(np.asarray(old_ids, np.uint64)) >> np.uint64(54)).astype(np.float32)
    return (base[:, None] + np.arange(dim, dtype=np.float32)[None, :]).astype(np.float16)


def test_features_f16_gpu(num_rows: int, dim: int, out: np.ndarray, device="cuda",
                          rows_per_chunk=1 << 21):
    """expected_rows_f16 for rows [0, num_rows), computed on the GPU and copied
    into `out` (pinned or registered host memory, num_rows*dim*2 bytes)."""
    import torch
    if isinstance(out, torch.Tensor):
        dst = out.view(torch.float16)[: num_rows * dim].view(num_rows, dim)
    else:
        dst = torch.from_numpy(out.reshape(-1)[: num_rows * dim * 2].view(np.float16)).view(num_rows, dim)
    cols = torch.arange(dim, dtype=torch.float32, device=device)
    for r0 in range(0, num_rows, rows_per_chunk):
        r1 = min(num_rows, r0 + rows_per_chunk)
        r = torch.arange(r0, r1, dtype=torch.int64, device=device)
        base = ((mix64_torch(r) >> 54) & 1023).to(torch.float32)
        dst[r0:r1].copy_((base[:, None] + cols[None, :]).to(torch.float16))
    torch.cuda.synchronize()
    return out
