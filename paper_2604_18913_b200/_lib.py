"""ctypes binding of the C ABI declared in include/th_b200.h.

The shared library is built in-tree (``paper_2604_18913_b200/lib/libth_b200.so``,
see ``__graft_entry__.build``).  There is no fallback: if the library or a
CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("TH_B200_LIB", Path(__file__).resolve().parent / "lib" / "libth_b200.so"))

(TH_OK, TH_ERR_INVALID, TH_ERR_RANGE, TH_ERR_CUDA, TH_ERR_NOMEM, TH_ERR_OVERFLOW, TH_ERR_STATE,
 TH_ERR_DATA) = range(8)
TH_EXACT, TH_FRONTIER, TH_CUMULATIVE = 0, 1, 2
TH_WANT_FRONTIERS, TH_WANT_ACTIVATED, TH_WANT_PATHS, TH_SINGLETON_SEEDS = 0x1, 0x2, 0x4, 0x8
TH_GRAPH_NO_REVERSE = 0x1
TH_PLAN_HASH, TH_PLAN_LPT = 0, 1
ABI_VERSION = 1

# every symbol include/th_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "th_abi_version", "th_last_error", "th_graph_create", "th_graph_create_lkg", "th_graph_destroy",
    "th_graph_info_get", "th_session_create", "th_session_destroy", "th_run", "th_finish",
    "th_session_set_pull_divisor", "th_session_launch_count", "th_plan_owner_hash",
    "th_session_set_list_min_entities", "th_session_set_overlap", "th_session_set_graphs", "th_session_set_dense_pull",
    "th_session_set_profiling", "th_session_profile", "th_session_profile_trace", "th_session_wave_lists",
    "th_shard_create", "th_shard_destroy", "th_shard_local_triples", "th_shard_launch_count",
    "th_shard_begin", "th_shard_can_pull", "th_shard_set_pull_divisor", "th_shard_region",
    "th_shard_ipc_handle", "th_shard_connect", "th_shard_ipc_open", "th_shard_grow_inbox",
    "th_shard_inbox_overflowed", "th_shard_hop", "th_shard_finish", "th_shard_sent", "th_shard_columns",
    "th_shard_hub_cache", "th_shard_hub_cache_stats", "th_shard_hub_cache_trace",
    "th_shard_hub_cache_resident", "th_shard_set_profiling", "th_shard_profile_trace",
    "th_shards_run_hops", "th_shards_run_wave",
    "th_ids_route_count", "th_ids_map_scatter", "th_ids_to_local_bits", "th_bits_andnot_update",
    "th_bits_or", "th_bits_compact", "th_plan_subjects", "th_session_set_k4_mode",
    "th_session_set_pull_screen", "th_session_wave_modes", "th_session_set_knob",
)
PROF_CATEGORIES = ("setup", "edges", "activated", "push", "pull", "frontier", "clear", "paths")

_c_i32p = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p


class GraphInfo(ctypes.Structure):
    _fields_ = [
        ("n_entities", ctypes.c_int64), ("n_triples", ctypes.c_int64), ("n_relations", ctypes.c_int64),
        ("indptr", _vp), ("csr_tid", _vp), ("csr_obj", _vp), ("csr_rel", _vp),
        ("subj", _vp), ("obj", _vp), ("rel", _vp),
        ("rindptr", _vp), ("rsrc", _vp), ("rrel", _vp),
        ("max_out_degree", ctypes.c_int64), ("max_in_degree", ctypes.c_int64),
        ("n_heavy_in", ctypes.c_int64), ("device_bytes", ctypes.c_uint64),
    ]


class Query(ctypes.Structure):
    _fields_ = [
        ("n_queries", ctypes.c_int32), ("d_seed_offsets", _vp), ("d_seeds", _vp),
        ("k", ctypes.c_int32), ("semantics", ctypes.c_int32),
        ("d_rel_masks", _vp), ("mask_words", ctypes.c_int32),
        ("flags", ctypes.c_uint32), ("max_paths", ctypes.c_int64),
    ]


class ShardCols(ctypes.Structure):
    _fields_ = [
        ("n_triples", ctypes.c_int64), ("n_local", ctypes.c_int64), ("n_hubs", ctypes.c_int64),
        ("subj_row", _vp), ("rel", _vp), ("obj", _vp), ("tid_l2g", _vp), ("l2g", _vp), ("hub_ids", _vp),
    ]


class Result(ctypes.Structure):
    _fields_ = [
        ("n_queries", ctypes.c_int32), ("k", ctypes.c_int32),
        ("frontier_off", _vp), ("frontier_len", _vp), ("frontier_ids", _vp),
        ("act_off", _vp), ("act_len", _vp), ("act_ids", _vp),
        ("edges", _vp),
        ("path_off", _vp), ("path_count", _vp), ("path_truncated", _vp), ("path_tids", _vp),
        ("frontier_total", ctypes.c_int64), ("act_total", ctypes.c_int64), ("path_total", ctypes.c_int64),
        ("push_hops", ctypes.c_int32), ("pull_hops", ctypes.c_int32),
    ]


_LIB = None


def load():
    """Load and type the library (raises if it was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"CUDA extension not built: {LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    sig = {
        "th_abi_version": (ctypes.c_int, []),
        "th_last_error": (ctypes.c_char_p, []),
        "th_graph_create": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_uint32, _vp, ctypes.POINTER(_vp)]),
        "th_graph_destroy": (ctypes.c_int, [_vp]),
        "th_graph_create_lkg": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int32, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32, _vp,
                                               ctypes.POINTER(_vp)]),
        "th_graph_info_get": (ctypes.c_int, [_vp, ctypes.POINTER(GraphInfo)]),
        "th_session_create": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(_vp)]),
        "th_session_destroy": (ctypes.c_int, [_vp]),
        "th_run": (ctypes.c_int, [_vp, ctypes.POINTER(Query)]),
        "th_finish": (ctypes.c_int, [_vp, ctypes.POINTER(Result)]),
        "th_session_set_pull_divisor": (ctypes.c_int, [_vp, ctypes.c_double]),
        "th_session_set_list_min_entities": (ctypes.c_int, [_vp, ctypes.c_int64]),
        "th_session_set_overlap": (ctypes.c_int, [_vp, ctypes.c_int]),
        "th_session_set_k4_mode": (ctypes.c_int, [_vp, ctypes.c_int]),
        "th_session_set_pull_screen": (ctypes.c_int, [_vp, ctypes.c_int]),
        "th_session_set_knob": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int64]),
        "th_session_set_graphs": (ctypes.c_int, [_vp, ctypes.c_int]),
        "th_session_set_dense_pull": (ctypes.c_int, [_vp, ctypes.c_double]),
        "th_session_launch_count": (ctypes.c_int64, [_vp]),
        "th_plan_owner_hash": (ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp]),
        "th_session_set_profiling": (ctypes.c_int, [_vp, ctypes.c_int]),
        "th_session_profile": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
        "th_session_wave_lists": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
        "th_session_wave_modes": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int32), ctypes.c_int]),
        "th_shard_create": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           _vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                           ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _vp,
                                           ctypes.POINTER(_vp)]),
        "th_shard_destroy": (ctypes.c_int, [_vp]),
        "th_shard_local_triples": (ctypes.c_int64, [_vp]),
        "th_shard_launch_count": (ctypes.c_int64, [_vp]),
        "th_shard_begin": (ctypes.c_int, [_vp, ctypes.POINTER(Query)]),
        "th_shard_can_pull": (ctypes.c_int, [_vp]),
        "th_shard_set_pull_divisor": (ctypes.c_int, [_vp, ctypes.c_double]),
        "th_shard_region": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_uint64),
                                           ctypes.POINTER(ctypes.c_int64)]),
        "th_shard_ipc_handle": (ctypes.c_int, [_vp, _vp]),
        "th_shard_connect": (ctypes.c_int, [_vp, ctypes.c_int32, _vp]),
        "th_shard_ipc_open": (ctypes.c_int, [_vp, ctypes.c_int32, _vp]),
        "th_shard_grow_inbox": (ctypes.c_int, [_vp, ctypes.c_int64]),
        "th_shard_inbox_overflowed": (ctypes.c_int, [_vp]),
        "th_shard_sent": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
        "th_shard_columns": (ctypes.c_int, [_vp, ctypes.POINTER(ShardCols)]),
        "th_shard_hop": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32]),
        "th_shard_finish": (ctypes.c_int, [_vp, ctypes.POINTER(Result)]),
        "th_session_profile_trace": (ctypes.c_int64, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int64]),
        "th_shard_hub_cache": (ctypes.c_int, [_vp, ctypes.c_int64]),
        "th_shard_set_profiling": (ctypes.c_int, [_vp, ctypes.c_int]),
        "th_shards_run_hops": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32]),
        "th_shards_run_wave": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.POINTER(Query),
                                              ctypes.POINTER(ctypes.c_int64)]),
        "th_shard_profile_trace": (ctypes.c_int64, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int64]),
        "th_shard_hub_cache_stats": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int64)]),
        "th_shard_hub_cache_trace": (ctypes.c_int64, [_vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]),
        "th_shard_hub_cache_resident": (ctypes.c_int64, [_vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]),
        "th_ids_route_count": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int32,
                                              _vp, _vp]),
        "th_ids_map_scatter": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp,
                                              ctypes.c_int64, _vp]),
        "th_ids_to_local_bits": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp, _vp]),
        "th_bits_andnot_update": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp]),
        "th_bits_or": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp]),
        "th_bits_compact": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                           ctypes.POINTER(ctypes.c_int64), _vp]),
        "th_plan_subjects": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _vp, _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.th_abi_version() != ABI_VERSION:
        raise RuntimeError("libth_b200.so ABI version mismatch; rebuild the extension")
    _LIB = lib
    return lib


def check(rc: int) -> None:
    """Map a status code to the reference's exception types."""
    if rc == TH_OK:
        return
    msg = load().th_last_error().decode(errors="replace")
    if rc in (TH_ERR_INVALID, TH_ERR_RANGE):
        raise ValueError(msg)
    if rc == TH_ERR_NOMEM:
        raise MemoryError(msg)
    if rc == TH_ERR_OVERFLOW:
        raise OverflowError(msg)
    if rc == TH_ERR_DATA:
        from .errors import ArchiveError

        raise ArchiveError(msg)
    raise RuntimeError(f"th_b200 error {rc}: {msg}")


class DeviceArray:
    """Zero-copy __cuda_array_interface__ view of library-owned memory."""

    def __init__(self, ptr: int, shape: tuple, typestr: str, owner=None):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(ptr or 0), False), "version": 3, "strides": None, "stream": None,
        }


def as_tensor(ptr: int, shape: tuple, typestr: str, owner=None):
    import torch

    n = 1
    for s in shape:
        n *= int(s)
    if n == 0 or not ptr:
        dt = {"<i4": torch.int32, "<i8": torch.int64, "|u1": torch.uint8, "<i2": torch.int16}[typestr]
        return torch.empty(tuple(int(s) for s in shape), dtype=dt, device="cuda")
    return torch.as_tensor(DeviceArray(ptr, shape, typestr, owner), device="cuda")
