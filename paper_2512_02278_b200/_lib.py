"""ctypes binding of libdvsg.so -- the C-ABI declared in include/dvsg.h.

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared object is missing this module raises at
import time, so no caller can silently run anything but the CUDA path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# DVSG_LIB selects a build variant (scripts/build_variant.sh) for A/B measurements
LIB_PATH = os.environ.get("DVSG_LIB") or os.path.join(_HERE, "libdvsg.so")

if not os.path.isfile(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the B200 search path has no CPU fallback)")

lib = ctypes.CDLL(LIB_PATH)

DVSG_OK, DVSG_EINVAL, DVSG_EFORMAT, DVSG_EINTERNAL = 0, 2, 3, 4
METRIC_L2, METRIC_IP = 0, 1
ACCUM_F64, ACCUM_F32, ACCUM_F32C = 0, 1, 2
RANGE_EXCLUDE_SELF, RANGE_BUILD_PAD, RANGE_MERGE, RANGE_OUT_PHYSICAL = 1, 2, 4, 8
COMMIT_ENTRY_ORDER, COMMIT_IOTA_IDS = 1, 2


class dvsg_search_params(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("beam_width", c_int), ("k", c_int),
                ("entry_count", c_int), ("metric", c_int), ("accum", c_int)]


P_u32 = POINTER(c_uint32)
P_f32 = POINTER(c_float)
P_u64 = POINTER(c_uint64)
P_params = POINTER(dvsg_search_params)

_SIGS = {
    "dvsg_last_error": (c_char_p, []),
    "dvsg_version": (c_char_p, []),
    "dvsg_create": (c_int, [c_int, POINTER(c_void_p)]),
    "dvsg_destroy": (c_int, [c_void_p]),
    "dvsg_stream": (c_void_p, [c_void_p]),
    "dvsg_synchronize": (c_int, [c_void_p]),
    "dvsg_index_reset": (c_int, [c_void_p]),
    "dvsg_set_centroids": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_int]),
    "dvsg_load_partition": (c_int, [c_void_p, c_uint32, c_uint64, c_int, c_int, c_void_p,
                                    c_void_p, c_void_p, c_void_p]),
    "dvsg_load_index_file": (c_int, [c_void_p, c_char_p, c_int]),
    "dvsg_save_index_file": (c_int, [c_char_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                                     c_void_p, c_void_p, c_void_p, c_void_p]),
    "dvsg_index_info": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_int),
                                POINTER(c_int), c_void_p, c_void_p]),
    "dvsg_get_entry_order": (c_int, [c_void_p, c_uint32, c_void_p]),
    "dvsg_compute_entry_order": (c_int, [c_void_p, c_uint64, c_int, c_void_p]),
    "dvsg_beam_search": (c_int, [c_void_p, c_uint32, c_void_p, c_uint64, c_int, P_params,
                                 c_void_p, c_void_p, c_void_p, c_void_p]),
    "dvsg_search_units_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_void_p, c_void_p,
                                         c_uint64, P_params, c_void_p, c_void_p, c_void_p,
                                         c_void_p]),
    "dvsg_beam_search_sharded_emulated": (c_int, [c_void_p, c_int, c_void_p, c_uint64, c_int, P_params,
                                                  c_void_p, c_void_p, c_void_p, c_void_p]),
    "dvsg_shard_init": (c_int, [c_void_p, c_int, c_int, c_uint64, c_int, c_int, c_void_p, c_void_p,
                                c_void_p, c_void_p]),
    "dvsg_shard_init_resident": (c_int, [c_void_p, c_int, c_int]),
    "dvsg_shard_export": (c_int, [c_void_p, c_void_p]),
    "dvsg_shard_connect": (c_int, [c_void_p, c_void_p]),
    "dvsg_shard_prepare": (c_int, [c_void_p]),
    "dvsg_search_sharded_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, P_params, c_void_p,
                                           c_void_p, c_void_p, c_void_p]),
    "dvsg_assign_top_c": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_int, c_void_p]),
    "dvsg_combine_results": (c_int, [c_void_p, c_uint64, c_int, c_void_p, c_void_p, c_void_p,
                                     c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "dvsg_run_pipeline": (c_int, [c_void_p, c_void_p, c_uint64, c_int, P_params, c_int, c_int,
                                  c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dvsg_run_pipeline_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, P_params, c_int,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dvsg_build_graph": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_int, c_void_p]),
    "dvsg_brute_force_topk": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_void_p, c_uint64, c_int,
                                      c_void_p, c_void_p]),
    "dvsg_assign_top_c_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_int, c_void_p]),
    "dvsg_combine_results_device": (c_int, [c_void_p, c_uint64, c_int, c_void_p, c_void_p, c_void_p,
                                            c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "dvsg_gather_vectors_device": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64, c_int, c_void_p]),
    "dvsg_set_shard_exchange": (c_int, [c_void_p, c_int]),
    "dvsg_nccl_unique_id": (c_int, [c_void_p, c_void_p]),
    "dvsg_nccl_connect": (c_int, [c_void_p, c_void_p]),
    "dvsg_set_timing": (c_int, [c_void_p, c_int]),
    "dvsg_last_pipeline_timeline": (c_int, [c_void_p, c_void_p, c_int, c_void_p]),
    "dvsg_last_sharded_timeline": (c_int, [c_void_p, c_void_p, c_int, c_void_p]),
    "dvsg_last_timings": (c_int, [c_void_p, P_f32, P_f32, P_f32, P_f32]),
    "dvsg_kernel_launches": (c_uint64, [c_void_p]),
    "dvsg_last_assign_info": (c_int, [c_void_p, c_void_p, c_void_p]),
    "dvsg_last_knn_info": (c_int, [c_void_p, c_void_p, c_void_p]),
    "dvsg_set_vector_storage": (c_int, [c_void_p, c_int]),
    "dvsg_last_search_stats": (c_int, [c_void_p, P_u64, P_u64, P_u64]),
    "dvsg_debug_counters": (c_int, [c_void_p, c_void_p]),
    "dvsg_row_norms_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_void_p]),
    "dvsg_range_topk_device": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                                       c_void_p, c_uint64, c_void_p, c_void_p, c_int, c_int, c_void_p,
                                       c_void_p, c_uint64]),
    "dvsg_to_bf16_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_int, c_void_p]),
    "dvsg_range_topk_bf16_device": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                                            c_void_p, c_uint64, c_void_p, c_void_p, c_int, c_int, c_void_p,
                                            c_void_p, c_uint64]),
    "dvsg_segment_means_device": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_uint32, c_void_p]),
    "dvsg_compute_entry_order_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_int, c_void_p]),
    "dvsg_partition_alloc_device": (c_int, [c_void_p, c_uint32, c_uint64, c_int, c_int, POINTER(c_void_p),
                                            POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p)]),
    "dvsg_partition_commit_device": (c_int, [c_void_p, c_int]),
    "dvsg_index_integral": (c_int, [c_void_p, POINTER(c_int)]),
    "dvsg_kmeans_train": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_int, c_int, c_uint64, c_void_p,
                                  POINTER(c_int), c_void_p]),
    "dvsg_partition_database": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_void_p, c_int, c_void_p]),
    "dvsg_cluster_comm_init": (c_int, [c_void_p, c_int, c_int, c_uint64, c_int, c_int, c_int]),
    "dvsg_cluster_comm_export": (c_int, [c_void_p, c_void_p]),
    "dvsg_cluster_comm_connect": (c_int, [c_void_p, c_void_p]),
    "dvsg_cluster_comm_arena": (c_void_p, [c_void_p]),
    "dvsg_cluster_comm_connect_local": (c_int, [c_void_p, c_void_p]),
    "dvsg_run_pipeline_cluster_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, P_params, c_int, c_void_p,
                                                 c_void_p, c_void_p, c_void_p, c_void_p]),
    "dvsg_cluster_comm_check": (c_int, [c_void_p]),
    "dvsg_optimize_graph_device": (c_int, [c_void_p, c_void_p, c_uint64, c_int, c_int]),
    "dvsg_partition_view_device": (c_int, [c_void_p, c_uint32, POINTER(c_void_p), POINTER(c_void_p),
                                           POINTER(c_void_p), POINTER(c_void_p), POINTER(c_uint64)]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class DvsError(RuntimeError):
    """Base class; ``code`` is the dvsg status (2/3/4, commands.cpp:355-361)."""

    code = DVSG_EINTERNAL


class InvalidArgument(DvsError, ValueError):
    """std::invalid_argument / config_error in the reference (exit code 2)."""

    code = DVSG_EINVAL


class FormatError(DvsError):
    """format_error in the reference (exit code 3)."""

    code = DVSG_EFORMAT


class InternalError(DvsError):
    """internal_error and every CUDA failure (exit code 4)."""

    code = DVSG_EINTERNAL


_BY_CODE = {DVSG_EINVAL: InvalidArgument, DVSG_EFORMAT: FormatError, DVSG_EINTERNAL: InternalError}


def check(status: int) -> None:
    if status != DVSG_OK:
        msg = lib.dvsg_last_error().decode("utf-8", "replace")
        raise _BY_CODE.get(status, InternalError)(msg)
