"""tiergraph on B200: the data-tiering hot path of arXiv 2111.05894.

Two hot paths, hand-written CUDA for sm_100a behind a C-ABI
(include/tg_capi.h, libtiergraph_b200.so):

* hotness predictor — bit-exact train-seeded reverse PageRank (fp64 CSR
  SpMV) and the hot-set / permutation selection (radix sort);
* tiered feature gather — hot rows in local HBM (sharded across GPUs and
  read by peer loads), cold rows in pinned host memory read by UVA
  zero-copy, with the reference's byte accounting.

`tiergraph` mirrors the reference API; `producers` binds the host-side
input producers; `synth` builds the synthetic inputs of the named shapes.
"""
from . import tiergraph  # noqa: F401  (loads libtiergraph_b200.so; raises if missing)

__all__ = ["tiergraph"]
