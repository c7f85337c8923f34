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

The CUDA library is loaded when `tiergraph` (or a module importing it) is
first imported, not by importing this package, so the bench's reference arm
can use the `synth` fixtures without loading libtiergraph_b200.so. Importing
`tiergraph` raises if the library is missing: there is no fallback.
"""
import importlib

__all__ = ["tiergraph", "producers", "distributed", "synth"]


def __getattr__(name):
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
