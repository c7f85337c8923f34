"""ctypes binding of the C-ABI in include/tg_capi.h (libtiergraph_b200.so).

The library is the only compute path: there is no CPU fallback. Importing
this module on a machine without the built library raises immediately;
creating a context without an sm_100a device raises from the library.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtiergraph_b200.so")

TG_OK = 0
TG_ERR_DOMAIN = 2
TG_ERR_FORMAT = 3
TG_ERR_IO = 4
TG_ERR_INTERNAL = 5
TG_MAX_DEVICES = 16
TG_COLD_REORDERED = 0
TG_COLD_INDIRECT = 1
TG_COLD_PAD128 = 2
TG_GATHER_BULK = 4
TG_GATHER_L2PF = 8
TG_GATHER_SPREAD = 16
TG_COLD_SPLIT_TAIL = 32
TG_GATHER_DYNAMIC = 64


class TgLayout(C.Structure):
    _fields_ = [("num_rows", C.c_uint64), ("local_boundary", C.c_uint64),
                ("multi_boundary", C.c_uint64), ("num_devices", C.c_uint32),
                ("feature_dim", C.c_uint64), ("elem_bytes", C.c_uint32)]


class TgReport(C.Structure):
    _fields_ = [("local_accesses", C.c_uint64), ("peer_accesses", C.c_uint64),
                ("host_accesses", C.c_uint64), ("local_bytes", C.c_uint64),
                ("peer_bytes", C.c_uint64), ("host_bytes", C.c_uint64)]


class TgLocation(C.Structure):
    _fields_ = [("tier", C.c_uint8), ("device", C.c_uint32), ("row_within_tier", C.c_uint64)]


vp = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
I32 = C.c_int
D = C.c_double
PL = C.POINTER(TgLayout)
PR = C.POINTER(TgReport)

# name -> (restype, argtypes); every symbol declared in include/tg_capi.h
SIGNATURES = {
    "tg_last_error": (C.c_char_p, []),
    "tg_version": (C.c_char_p, []),
    "tg_ctx_create": (I32, [I32, C.POINTER(vp)]),
    "tg_ctx_create_on_stream": (I32, [I32, vp, C.POINTER(vp)]),
    "tg_ctx_destroy": (I32, [vp]),
    "tg_ctx_sync": (I32, [vp]),
    "tg_ctx_trim": (I32, [vp]),
    "tg_memcpy_async": (I32, [vp, vp, vp, U64]),
    "tg_ctx_stream": (vp, [vp]),
    "tg_ctx_device": (I32, [vp]),
    "tg_default_device": (I32, []),
    "tg_device_count": (I32, []),
    "tg_device_list": (I32, [C.POINTER(I32), I32]),
    "tg_kernel_launches": (U64, []),
    "tg_graph_create": (I32, [vp, vp, vp, U64, U64, C.POINTER(vp)]),
    "tg_graph_destroy": (I32, [vp]),
    "tg_graph_num_nodes": (U64, [vp]),
    "tg_graph_num_edges": (U64, [vp]),
    "tg_graph_offsets32": (vp, [vp]),
    "tg_graph_targets32": (vp, [vp]),
    "tg_degree_score": (I32, [vp, vp, vp]),
    "tg_in_degrees": (I32, [vp, vp, vp]),
    "tg_reverse_pagerank": (I32, [vp, vp, U32, D, vp]),
    "tg_weighted_reverse_pagerank": (I32, [vp, vp, U32, D, vp, U64, vp]),
    "tg_pagerank_prepare_async": (I32, [vp, vp, vp, U64, vp, vp]),
    "tg_pagerank_step_async": (I32, [vp, vp, vp, D, vp, vp, vp, U64, U64, I32]),
    "tg_pagerank_step_peers_async": (I32, [vp, vp, vp, D, vp, vp, vp, U64, U64, I32, vp, vp, U32]),
    "tg_peer_barrier_async": (I32, [vp, vp, vp, U32, U32, vp]),
    "tg_score_ordering": (I32, [vp, vp, U64, vp]),
    "tg_permutation_from_scores": (I32, [vp, vp, U64, vp, vp]),
    "tg_validate_permutation": (I32, [vp, vp, U64]),
    "tg_invert": (I32, [vp, vp, U64, vp]),
    "tg_reorder_features": (I32, [vp, vp, U64, U64, vp, U64, vp]),
    "tg_reorder_graph": (I32, [vp, vp, vp, U64, U64, vp, U64, vp, vp]),
    "tg_validate_layout": (I32, [PL]),
    "tg_validate_cost_model": (I32, [D, D, D]),
    "tg_resolve": (I32, [PL, U64, U32, C.POINTER(TgLocation)]),
    "tg_plan_layout": (I32, [U64, D, D, U32, U64, U32, U64, PL]),
    "tg_report_hit_ratio": (D, [PR]),
    "tg_report_est_transfer_seconds": (D, [PR, D, D, D]),
    "tg_gather_account": (I32, [vp, PL, vp, U64, U32, PR]),
    "tg_simulate_trace": (I32, [vp, vp, U64, PL, PR]),
    "tg_counts_in_row_order": (I32, [vp, vp, U64, vp, U64, vp]),
    "tg_hot_fraction_sweep": (I32, [vp, vp, U64, vp, vp, U64, D, U32, U64, U32, U64, PL, PR, vp]),
    "tg_store_create": (I32, [vp, PL, U32, U32, C.POINTER(vp)]),
    "tg_store_destroy": (I32, [vp]),
    "tg_store_place": (I32, [vp, vp, vp]),
    "tg_store_local_base": (vp, [vp]),
    "tg_store_local_rows": (U64, [vp]),
    "tg_store_cold_host_bytes": (U64, [vp]),
    "tg_store_set_peer": (I32, [vp, U32, vp]),
    "tg_store_share_cold": (I32, [vp, vp]),
    "tg_store_cold_tier_bytes": (U64, [vp]),
    "tg_store_attach_cold": (I32, [vp, vp, U64, I32]),
    "tg_host_shared_map": (I32, [C.c_char_p, U64, I32, C.POINTER(vp)]),
    "tg_host_shared_unmap": (I32, [vp, U64]),
    "tg_host_shared_unlink": (I32, [C.c_char_p]),
    "tg_gather_rows": (I32, [vp, vp, U64, vp, PR]),
    "tg_gather_rows_async": (I32, [vp, vp, U64, vp, vp, vp]),
    "tg_enable_peer_access": (I32, [I32, I32]),
    "tg_ipc_get_handle": (I32, [vp, vp]),
    "tg_ipc_open_handle": (I32, [vp, vp, C.POINTER(vp)]),
    "tg_ipc_close_handle": (I32, [vp]),
    "tg_measure_host_rows_us": (I32, [vp, vp, U64, U64, U64, U64, C.c_int, C.POINTER(C.c_double)]),
    "tg_store_measure_cold_us": (I32, [vp, U64, C.c_int, C.POINTER(C.c_double)]),
    "tg_store_measure_cold_rows_us": (I32, [vp, U64, C.c_int, C.POINTER(C.c_double)]),
    "tg_mapped_device_ptr": (vp, [vp]),
    "tg_store_place_rows": (I32, [vp, vp, U64, vp]),
    "tg_time_gather_rows": (I32, [vp, vp, vp, U64, vp, C.c_int, vp, C.POINTER(C.c_double)]),
    "tg_graph_load_csrg": (I32, [vp, C.c_char_p, C.POINTER(vp)]),
    "tg_store_place_feat": (I32, [vp, C.c_char_p, vp]),
    "tg_transpose": (I32, [vp, vp, vp, U64, U64, vp, vp]),
    "tg_sample_batches": (I32, [vp, vp, U64, U64, U64, U64, vp, U32, U64, U64, vp, U64, vp]),
    "tg_device_alloc": (I32, [vp, U64, C.POINTER(vp)]),
    "tg_device_free": (I32, [vp, vp]),
    "tg_host_register": (I32, [vp, U64]),
    "tg_host_unregister": (I32, [vp]),
    "tg_host_alloc": (I32, [U64, C.POINTER(vp)]),
    "tg_host_free": (I32, [vp]),
    "tg_measure_host_read_gbps": (I32, [vp, U64, U64, I32, C.POINTER(D)]),
    "tg_measure_hbm_copy_gbps": (I32, [vp, U64, I32, C.POINTER(D)]),
    "tg_host_last_error": (C.c_char_p, []),
    "tg_free": (None, [vp]),
    "tg_draw_random_train_ids": (I32, [U64, U64, U64, vp]),
    "tg_transpose_host": (I32, [vp, vp, U64, vp, vp]),
    "tg_epoch_minibatches": (I32, [vp, vp, U64, vp, U64, vp, U32, U64, U64, U64, U64, U64, I32,
                                   C.POINTER(vp), C.POINTER(U64), C.POINTER(vp)]),
    "tg_measure_gather_floor_us": (I32, [vp, vp, I32, C.POINTER(D)]),
    "tg_weighted_reverse_pagerank_timed": (I32, [vp, vp, U32, D, vp, U64, vp, vp]),
    "tg_row_blocks": (I32, [vp, U64, U32, vp]),
    "tg_graph_create_rows": (I32, [vp, vp, vp, U64, U64, U64, U64, C.POINTER(vp)]),
    "tg_graph_row_range": (I32, [vp, C.POINTER(U64), C.POINTER(U64)]),
    "tg_in_degrees_u32_async": (I32, [vp, vp, vp]),
    "tg_pagerank_init_async": (I32, [vp, U64, vp, U64, vp, vp]),
    "tg_mgraph_create": (I32, [vp, U32, vp, vp, U64, U64, C.POINTER(vp)]),
    "tg_mgraph_destroy": (I32, [vp]),
    "tg_mgraph_info": (I32, [vp, vp, vp, C.POINTER(D)]),
    "tg_mgraph_in_degrees": (I32, [vp, vp]),
    "tg_mgraph_pagerank": (I32, [vp, U32, D, vp, U64, I32, vp]),
    "tg_pagerank_relabel_info": (I32, [vp, vp, C.POINTER(I32), C.POINTER(D)]),
    "tg_sampler_create": (I32, [vp, vp, C.POINTER(vp)]),
    "tg_sgraph_cold_bytes": (U64, [vp, U64, PL]),
    "tg_sgraph_create": (I32, [vp, PL, U32, vp, vp, U64, U64, vp, U64, I32, C.POINTER(vp)]),
    "tg_sgraph_destroy": (I32, [vp]),
    "tg_sgraph_local_base": (vp, [vp]),
    "tg_sgraph_set_peer": (I32, [vp, U32, vp]),
    "tg_sgraph_cold_host": (vp, [vp]),
    "tg_sgraph_info": (I32, [vp, vp]),
    "tg_sampler_create_tiered": (I32, [vp, vp, C.POINTER(vp)]),
    "tg_sampler_structure_reads": (I32, [vp, vp, I32]),
    "tg_sampler_destroy": (I32, [vp]),
    "tg_sample_minibatch": (I32, [vp, vp, U64, vp, U32, U64, U64, U64, vp, U64, C.POINTER(U64)]),
    "tg_epoch_order": (I32, [vp, U64, U64, U64, vp]),
    "tg_sample_minibatch_raw": (I32, [vp, vp, U64, vp, U32, U64, U64, U64, vp, U64,
                                      C.POINTER(U64), vp, U64, C.POINTER(U64)]),
    "tg_sampler_trace": (I32, [vp, vp, U64, vp, U32, U64, U64, U64, I32, vp]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(tiergraph_b200 has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = load()
