"""Seeded fixtures shared by the tests (test infrastructure, not product).

Pure-Python copies of the reference test helpers so fixtures are identical:
``RngStream`` (rng.hpp:32-59), ``random_graph`` (tests/test_helpers.hpp:15-28),
``random_permutation`` (tests/test_reorder.cpp:29-36), ``random_counter``
(tests/test_tiering.cpp:26-33) and ``dense_reverse_pagerank``
(tests/oracles.hpp:18-52).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def derive_stream_key(seed: int, coords) -> int:
    h = mix64(seed ^ 0x6A09E667F3BCC908)
    for c in coords:
        h = mix64(h ^ mix64(c))
    return h


class RngStream:
    def __init__(self, key: int):
        self.state = key & M64

    def next_u64(self) -> int:
        v = mix64(self.state)
        self.state = (self.state + 1) & M64
        return v

    def next_below(self, bound: int) -> int:
        x = self.next_u64()
        m = x * bound
        lo = m & M64
        if lo < bound:
            threshold = ((1 << 64) - bound) % bound
            while lo < threshold:
                x = self.next_u64()
                m = x * bound
                lo = m & M64
        return m >> 64

    def next_unit(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53


def random_graph(oracle, n: int, avg_degree: float, seed: int, allow_self_loops=True):
    rng = RngStream(derive_stream_key(seed, [0x7267]))
    m = int(avg_degree * n)
    src, dst = [], []
    for _ in range(m):
        s = rng.next_below(n)
        d = rng.next_below(n)
        if not allow_self_loops and s == d:
            continue
        src.append(s)
        dst.append(d)
    return oracle.from_edge_list(n, np.array(src, np.uint64), np.array(dst, np.uint64))


def graph_from_pairs(oracle, n, pairs):
    src = np.array([p[0] for p in pairs], np.uint64)
    dst = np.array([p[1] for p in pairs], np.uint64)
    return oracle.from_edge_list(n, src, dst)


def random_permutation(n: int, seed: int, tag: int = 0x70) -> np.ndarray:
    perm = list(range(n))
    rng = RngStream(derive_stream_key(seed, [tag]))
    for i in range(n, 1, -1):
        j = rng.next_below(i)
        perm[i - 1], perm[j] = perm[j], perm[i - 1]
    return np.array(perm, np.uint64)


def random_counter(n: int, seed: int, tag: int = 0x63, bound: int = 20) -> np.ndarray:
    rng = RngStream(derive_stream_key(seed, [tag]))
    c = np.array([rng.next_below(bound) for _ in range(n)], np.uint64)
    if not c.any():
        c[0] = 1
    return c


def random_layout(rng: RngStream, n: int):
    mb = rng.next_below(n + 1)
    lb = rng.next_below(mb + 1)
    d = 1 + rng.next_below(6)
    dim = 1 + rng.next_below(64)
    eb = 4 if rng.next_below(2) == 0 else 8
    return (n, lb, mb, d, dim, eb)


def dense_reverse_pagerank(off, tgt, iterations=5, damp=0.85, labeled=None):
    n = len(off) - 1
    adj = np.zeros((n, n), np.uint8)
    for u in range(n):
        for v in tgt[off[u]:off[u + 1]]:
            adj[u, v] = 1
    indeg = np.maximum(adj.sum(axis=0).astype(np.float64), 1.0)
    score = np.full(n, 1.0 / n)
    if labeled is not None and len(labeled):
        w = n / len(labeled)
        for i in labeled:
            score[i] *= w
    base = (1.0 - damp) / n
    for _ in range(iterations):
        norm = score / indeg
        nxt = np.empty(n)
        for j in range(n):
            pulled = 0.0
            for v in np.nonzero(adj[j])[0]:
                pulled += norm[v]
            nxt[j] = base + damp * pulled
        score = nxt
    return score
