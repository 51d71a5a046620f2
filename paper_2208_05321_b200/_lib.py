"""ctypes binding of libfreqcache_b200.so (C ABI in include/freqcache_b200.h).

The library is built in-tree (`python -m paper_2208_05321_b200.build`). There is
no CPU fallback: if the library is missing or no CUDA device is present, every
cache verb raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int32, c_int64, c_uint64, c_void_p

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfreqcache_b200.so")
# A/B measurements only: another in-tree build of the same ABI (tools/build_ab.sh)
LIB_PATH = os.environ.get("FC_LIB_PATH", LIB_PATH)

# fc_status (include/freqcache_b200.h)
OK = 0
ERR_BATCH_EXCEEDS_CAPACITY = 1
ERR_ID_OUT_OF_RANGE = 2
ERR_INSUFFICIENT_EVICTABLE = 3
ERR_INSUFFICIENT_FREE_SLOTS = 4
ERR_BUFFER_TOO_SMALL = 5
ERR_CUDA = 6
ERR_BAD_ARG = 7
ERR_SLOT_OUT_OF_RANGE = 8
ERR_NOT_EMPTY = 9
ERR_NO_SLOW_TIER = 10

IPC_HANDLE_BYTES = 128  # FC_IPC_HANDLE_BYTES

WB = {"dirty_only": 0, "always": 1}
EVICT = {"occupancy_aware": 0, "paper_literal": 1}
POOL = {"sum": 0, "mean": 1}
OPTIM = {"sgd": 0, "adagrad": 1}


class PrepareInfo(ctypes.Structure):
    _fields_ = [("unique", c_int64), ("hits", c_int64), ("misses", c_int64), ("evictions", c_int64),
                ("rows_to_slow", c_int64), ("free_count", c_int64), ("bad_id", c_int64),
                ("candidates", c_int64)]


class Views(ctypes.Structure):
    _fields_ = [("fast_rows", c_void_p), ("slot_to_rank", c_void_p), ("rank_to_slot", c_void_p),
                ("dirty", c_void_p), ("rank_of", c_void_p), ("fast_state", c_void_p),
                ("capacity", c_int64), ("num_ids", c_int64), ("dim", c_int64), ("state_width", c_int64)]


_SIGS = {
    "fc_create": (c_int32, [c_int64, c_int64, c_int32, c_int32, c_int32, c_int32, c_int64, c_int32, POINTER(c_void_p)]),
    "fc_destroy": (c_int32, [c_void_p]),
    "fc_last_error": (c_char_p, []),
    "fc_get_views": (c_int32, [c_void_p, POINTER(Views)]),
    "fc_host_alloc": (c_int32, [c_int64, POINTER(c_void_p)]),
    "fc_host_free": (c_int32, [c_void_p]),
    "fc_set_idx_map": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "fc_attach_slow_tier": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int64]),
    "fc_set_modes": (c_int32, [c_void_p, c_int32, c_int32]),
    "fc_free_count": (c_int64, [c_void_p]),
    "fc_set_buffer_bytes": (c_int32, [c_void_p, c_int64]),
    "fc_profile": (c_int32, [c_void_p, c_int32, c_void_p]),
    "fc_set_engine": (c_int32, [c_void_p, c_int32]),
    "fc_drain": (c_int32, [c_void_p]),
    "fc_drain_stream": (c_int32, [c_void_p, c_void_p]),
    "fc_warmup": (c_int32, [c_void_p, c_int64, c_void_p]),
    "fc_prepare": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_void_p, c_void_p, POINTER(PrepareInfo)]),
    "fc_prepare_begin": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p]),
    "fc_prepare_commit": (c_int32, [c_void_p, c_void_p, POINTER(PrepareInfo)]),
    "fc_last_writebacks": (c_int32, [c_void_p, POINTER(c_int64)]),
    "fc_memory_bytes": (c_int32, [c_void_p, POINTER(c_int64), c_int32]),
    "fc_build_reorder": (c_int32, [c_void_p, c_int32, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                   POINTER(c_int64), c_void_p]),
    "fc_router_create": (c_int32, [c_int64, c_int32, c_int32, POINTER(c_void_p)]),
    "fc_router_create_tables": (c_int32, [c_int64, c_int32, c_int32, c_void_p, c_void_p, c_int32, POINTER(c_void_p)]),
    "fc_router_destroy": (c_int32, [c_void_p]),
    "fc_route": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_void_p, POINTER(c_int64),
                           c_void_p]),
    "fc_pool_rows": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_int32, c_int64, c_int32, c_void_p,
                               c_int32, c_void_p, c_void_p]),
    "fc_route_grads": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_int32, c_void_p,
                                 c_int32, c_void_p, c_int32, c_void_p, c_void_p]),
    "fc_pool_to_peers": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                   c_void_p]),
    "fc_gather_from_peers": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_int32, c_void_p, c_void_p]),
    "fc_pool_cols_to_peers": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                        c_int64, c_int64, c_void_p, c_void_p]),
    "fc_gather_cols_from_peers": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_int32, c_int64, c_int64,
                                            c_void_p, c_void_p]),
    "fc_ipc_handle": (c_int32, [c_void_p, c_void_p]),
    "fc_ipc_open": (c_int32, [c_void_p, c_int32, POINTER(c_void_p)]),
    "fc_ipc_close": (c_int32, [c_void_p]),
    "fc_trace": (c_int32, [c_void_p, c_int32]),
    "fc_trace_mark": (c_int32, [c_void_p, c_int32, c_void_p]),
    "fc_trace_read": (c_int64, [c_void_p, c_void_p, c_void_p, c_int64]),
    "fc_last_events": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "fc_flush": (c_int32, [c_void_p, c_void_p, POINTER(c_int64)]),
    "fc_mark_dirty": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    "fc_select_evictions": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p]),
    "fc_pooled_forward": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int32, c_int64, c_int32,
                                    c_void_p, c_int32, c_void_p, c_void_p]),
    "fc_gather_rows": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fc_apply_unique_update": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fc_apply_synthetic_update": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_uint64, c_void_p,
                                            c_void_p]),
    "fc_scatter_update": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "fc_backward_update": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int32,
                                     c_int64, c_int32, c_void_p, c_int32, c_void_p, c_int32, c_float, c_float,
                                     c_void_p]),
}

EXPORTS = tuple(_SIGS)

_lib = None


def load():
    """Load the library once; raise loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2208_05321_b200.build` "
            "(the cache has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        if "FC_LIB_PATH" in os.environ and not hasattr(lib, name):
            continue  # an older A/B build may lack newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().fc_last_error()
    return msg.decode() if msg else ""
