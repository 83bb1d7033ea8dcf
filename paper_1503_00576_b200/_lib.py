"""ctypes binding of libtcb200.so (the C ABI in include/tricount_b200.h).

There is no CPU fallback: if the library or a B200 is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TC_LIB_PATH: development override (A/B of compile-time variants)
LIB_PATH = os.environ.get("TC_LIB_PATH") or os.path.join(_HERE, "libtcb200.so")

ALGO_AUTO = 0
ALGO_MERGE_THREAD = 1
PREPROCESS_RANK_SPACE = 1


ABI_VERSION = 3  # include/tricount_b200.h TC_ABI_VERSION


class TcTimes(ctypes.Structure):
    _fields_ = [
        ("h2d_ms", ctypes.c_double),
        ("preprocess_ms", ctypes.c_double),
        ("count_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("classify_ms", ctypes.c_double),
        ("heavy_ms", ctypes.c_double),
        ("light_ms", ctypes.c_double),
        ("heavy_tasks", ctypes.c_uint64),
        ("vmajor_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class TcError(RuntimeError):
    """A CUDA / library failure inside libtcb200 (argument errors raise ValueError)."""


_u32p = ctypes.POINTER(ctypes.c_uint32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p
_graph_p = ctypes.c_void_p

_SIGS = {
    "tc_init": ([ctypes.c_int], ctypes.c_int),
    "tc_shutdown": ([], ctypes.c_int),
    "tc_last_error": ([], ctypes.c_char_p),
    "tc_abi_version": ([], ctypes.c_int),
    "tc_preprocess": ([_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                       ctypes.POINTER(_graph_p), ctypes.POINTER(TcTimes)], ctypes.c_int),
    "tc_graph_upload": ([_vp, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64,
                         ctypes.POINTER(_graph_p)], ctypes.c_int),
    "tc_graph_create": ([ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(_graph_p)],
                        ctypes.c_int),
    "tc_graph_flags": ([_graph_p, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tc_preprocess_ex": ([_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                          ctypes.POINTER(_graph_p), ctypes.POINTER(TcTimes)], ctypes.c_int),
    "tc_graph_finalize": ([_graph_p], ctypes.c_int),
    "tc_graph_download": ([_graph_p, _vp, _vp, _vp], ctypes.c_int),
    "tc_graph_info": ([_graph_p, _u64p, _u64p, ctypes.POINTER(ctypes.c_uint32)], ctypes.c_int),
    "tc_graph_device_ptrs": ([_graph_p, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp)], ctypes.c_int),
    "tc_graph_free": ([_graph_p], ctypes.c_int),
    "tc_count": ([_graph_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _u64p,
                  ctypes.POINTER(TcTimes)], ctypes.c_int),
    "tc_count_partitioned": ([_graph_p, _vp, ctypes.c_int, ctypes.c_int, _u64p,
                              ctypes.POINTER(TcTimes)], ctypes.c_int),
    "tc_intersect_count": ([_graph_p, ctypes.c_uint32, ctypes.c_uint32, _u64p], ctypes.c_int),
    "tc_count_with_timings": ([_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                               _u64p, ctypes.POINTER(TcTimes)], ctypes.c_int),
    "tc_work_bounds": ([_graph_p, ctypes.c_int, _vp], ctypes.c_int),
    "tc_merge_work": ([_graph_p, _u64p], ctypes.c_int),
    "tc_shard_plan": ([_graph_p, ctypes.c_int, _vp, _vp], ctypes.c_int),
    "tc_shard_cost_sizes": ([_graph_p, ctypes.c_int, _u64p, _u64p, _u64p, ctypes.POINTER(ctypes.c_uint32)],
                            ctypes.c_int),
    "tc_shard_costs": ([_graph_p, ctypes.c_int, _vp, _vp], ctypes.c_int),
    "tc_shard_stats": ([_graph_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _vp],
                       ctypes.c_int),
    "tc_count_shard": ([_graph_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _u64p,
                        ctypes.POINTER(TcTimes)], ctypes.c_int),
    "tc_sort_edges": ([_vp, ctypes.c_uint64, ctypes.c_uint64, _vp], ctypes.c_int),
    "tc_build_node_array": ([_vp, ctypes.c_uint64, ctypes.c_uint64, _vp], ctypes.c_int),
    "tc_orient_and_compact": ([_vp, ctypes.c_uint64, _vp, ctypes.c_uint64, _vp, _u64p],
                              ctypes.c_int),
    "tc_gen_rmat": ([ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), _u64p, _u64p,
                     ctypes.POINTER(_vp), _u64p, _u64p], ctypes.c_int),
    "tc_gen_ba": ([ctypes.c_uint64, ctypes.c_uint32, _u64p, _u64p, ctypes.POINTER(_vp), _u64p, _u64p],
                  ctypes.c_int),
    "tc_dist_degrees": ([_vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, _vp], ctypes.c_int),
    "tc_dist_orient": ([_vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, _vp, ctypes.POINTER(_vp),
                        _u64p, _vp], ctypes.c_int),
    "tc_dist_layout": ([_graph_p, _vp, ctypes.c_int, _vp, _vp], ctypes.c_int),
    "tc_dist_split": ([_vp, ctypes.c_uint64, ctypes.c_uint64, _vp, ctypes.c_int, _vp], ctypes.c_int),
    "tc_dist_place": ([_graph_p, _vp, ctypes.c_uint64, ctypes.c_uint64], ctypes.c_int),
    "tc_gen_rgg": ([ctypes.c_uint64, ctypes.c_double, _u64p, _u64p, ctypes.POINTER(_vp), _u64p, _u64p],
                   ctypes.c_int),
    "tc_read_tri1": ([ctypes.c_char_p, ctypes.POINTER(_vp), _u64p], ctypes.c_int),
    "tc_parse_edge_list": ([ctypes.c_char_p, ctypes.POINTER(_vp), _u64p, _u64p,
                            ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tc_validate_edge_array": ([_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                ctypes.POINTER(ctypes.c_int), _u64p], ctypes.c_int),
    "tc_wedge_count": ([_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, _u64p,
                        ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tc_device_alloc": ([ctypes.c_uint64, ctypes.POINTER(_vp)], ctypes.c_int),
    "tc_device_free": ([_vp], ctypes.c_int),
    "tc_memcpy": ([_vp, _vp, ctypes.c_uint64, ctypes.c_int], ctypes.c_int),
    "tc_host_alloc": ([ctypes.c_uint64, ctypes.POINTER(_vp)], ctypes.c_int),
    "tc_host_free": ([_vp], ctypes.c_int),
    "tc_host_register": ([_vp, ctypes.c_uint64], ctypes.c_int),
    "tc_host_unregister": ([_vp], ctypes.c_int),
    "tc_synchronize": ([], ctypes.c_int),
    "tc_l2_flush": ([], ctypes.c_int),
    "tc_timer_record": ([ctypes.c_int], ctypes.c_int),
    "tc_timer_elapsed": ([ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tc_launch_count": ([_u64p], ctypes.c_int),
    "tc_reserve": ([ctypes.c_uint64], ctypes.c_int),
    "tc_schedule_bytes": ([_graph_p, _vp], ctypes.c_int),
    "tc_schedule_bytes_range": ([_graph_p, ctypes.c_int64, ctypes.c_int64, _vp], ctypes.c_int),
    "tc_set_option": ([ctypes.c_char_p, ctypes.c_int64], ctypes.c_int),
    "tc_get_option": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "tc_reset_options": ([], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None
_initialised = False


def load(init: bool = False):
    """Load libtcb200.so (raises if absent); with init=True also bind the GPU."""
    global _lib, _initialised
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            if lib.tc_abi_version() != ABI_VERSION:  # TcTimes layout and signatures below
                raise ImportError(f"{LIB_PATH} has ABI {lib.tc_abi_version()}, this binding expects "
                                  f"{ABI_VERSION}: rebuild with `python __graft_entry__.py build`")
            _lib = lib
        if init and not _initialised:
            dev = int(os.environ.get("LOCAL_RANK", "0")) if "TC_DEVICE" not in os.environ \
                else int(os.environ["TC_DEVICE"])
            _check(_lib.tc_init(dev))
            _initialised = True
    return _lib


def lib():
    return load(init=True)


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (_lib.tc_last_error() or b"").decode(errors="replace")
    if rc == -1:
        raise ValueError(msg)
    if rc == -3:
        raise MemoryError(msg)
    if rc == -4:
        raise OSError(msg)
    raise TcError(msg)


def check(rc: int) -> None:
    _check(rc)


def set_option(name: str, value: int) -> None:
    """Schedule option (include/tricount_b200.h tc_set_option); tests and probes only."""
    _check(lib().tc_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    v = ctypes.c_int64()
    _check(lib().tc_get_option(name.encode(), ctypes.byref(v)))
    return v.value


def reset_options() -> None:
    _check(lib().tc_reset_options())


class options:
    """Context manager: `with options(vmajor=1, light=2): ...` (restores the defaults)."""

    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        for k, v in self.kv.items():
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        reset_options()


def ptr(arr: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(arr.ctypes.data) if arr.size else ctypes.c_void_p(0)
