"""ctypes binding of libgq_b200.so (the C-ABI in include/gq_b200.h).

There is no fallback: if the sm_100a library is missing or fails to load,
every entry point raises. Build it with `python -m paper_2305_18627_b200.build`
(or `__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("GQ_B200_LIB") or Path(__file__).resolve().parent / "libgq_b200.so")

GQ_OK, GQ_ERR_INVALID, GQ_ERR_OVERFLOW, GQ_ERR_DOMAIN, GQ_ERR_RUNTIME, GQ_ERR_CUDA = 0, 1, 2, 3, 4, 6
GQ_NORM_INF = 0xFFFFFFFF
GQ_NORM_L2_SEQUENTIAL = 0x102
GQ_OPT_QUANT_CTAS_PER_SM, GQ_OPT_REDUCE_CTAS_PER_SM, GQ_OPT_COMM_WAIT, GQ_OPT_PDL = 1, 2, 3, 4
GQ_OPT_COMM_TIMEOUT_S = 5
GQ_OPT_SMALL_PATH = 6
GQ_OPT_COMM_FOLD = 7
GQ_OPT_FUSED_PATH = 8
GQ_DTYPE_F32, GQ_DTYPE_F64 = 0, 1
GQ_MAX_WORKERS = 128

# Every symbol include/gq_b200.h declares, with its ctypes signature.
_u32, _u64, _i32, _vp, _f32 = C.c_uint32, C.c_uint64, C.c_int, C.c_void_p, C.c_float
_pp = C.POINTER(C.c_void_p)


class GqConfig(C.Structure):
    _fields_ = [("workers", _u32), ("kind", _u32), ("s", _u32), ("norm_q", _u32),
                ("norm_p", _u32), ("width_bits", _u32), ("topo", _u32), ("reserved", _u32),
                ("seed", _u64)]


class GqKdraws(C.Structure):
    _fields_ = [("buf", _vp), ("n", _u32), ("kind", _u32), ("width", _u32), ("s", _u32), ("topo", _u32),
                ("reserved", _u32), ("lane_begin", _u64), ("lane_end", _u64), ("seed", _u64), ("round", _u64)]


class GqPlan(C.Structure):
    _fields_ = [("lane_width", _u32), ("shift", _u32), ("m", _u32), ("max_e", _u32)]


class GqCommInfo(C.Structure):
    _fields_ = [("lane_width", _u32), ("n_local", _u32), ("worker_begin", _u32), ("host_wait", _u32),
                ("slice_lanes", _u64), ("lane_begin", _u64), ("lane_end", _u64), ("device", C.c_int32),
                ("reserved", _u32)]


SIGNATURES = {
    "gq_abi_version": (_i32, []),
    "gq_set_option": (_i32, [_u32, C.c_int64]),
    "gq_last_error": (C.c_char_p, []),
    "gq_plan_path": (_i32, [C.POINTER(GqConfig), C.POINTER(GqPlan)]),
    "gq_lane_bytes": (_u64, [_u64, _u32]),
    "gq_norm_workspace_bytes": (C.c_size_t, [_u32, _u64]),
    "gq_norm": (_i32, [_pp, _u32, _u32, _u64, _u32, _u32, _vp, _vp, _vp, _vp, _vp]),
    "gq_norm_combine": (_i32, [_vp, _u32, _u32, _u32, _vp, _vp]),
    "gq_quantize": (_i32, [_pp, _u32, _u32, C.POINTER(_u32), _u64, _vp, _u32, _u32, _u32, _u32,
                           _u64, _u64, _pp, _vp, _vp]),
    "gq_reduce_lanes": (_i32, [_pp, _u32, _u64, _u64, _u64, _u32, _u32, _u32, _u32, _u64, _u64,
                               _vp, _vp, _vp, _vp, _f32, _vp, _vp]),
    "gq_reduce_slice": (_i32, [_pp, _u32, _u64, _u64, _u64, _u32, _u32, _u32, _u32, _u64, _u64,
                               _vp, _vp, _vp, _vp, _f32, _vp, _vp]),
    "gq_combine_lanes": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _u32, _u32, _u64, _u64, _u32, _u32,
                                _vp, _vp]),
    "gq_rng_draws": (_i32, [_u64, _u64, _u64, _u64, _u64, _u64, _u32, _vp, _vp, _vp, _vp, _vp]),
    "gq_sparse_payload_bytes": (_u64, [_u64, _u32]),
    "gq_sparse_workspace_bytes": (C.c_size_t, [_u64]),
    "gq_sparse_encode": (_i32, [_vp, _u64, _u32, _u32, _u32, _u32, _vp, _vp, _vp, _vp, _vp]),
    "gq_sparse_mean_inproc": (_i32, [_pp, _u32, _u64, _u32, _u32, _u32, _vp, _vp, _vp, _vp]),
    "gq_sparse_accumulate": (_i32, [_vp, _u64, _u32, _u32, _u32, _u64, _vp, _vp, _vp]),
    "gq_sparse_finish": (_i32, [_vp, _u64, _u32, _vp, _vp, _vp, _f32, _vp]),
    "gq_dequant_f64": (_i32, [_vp, _u64, _u64, _vp, _u32, _u32, _u32, _u32, _vp, _vp, _vp]),
    "gq_malloc": (_i32, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "gq_free": (_i32, [_vp]),
    "gq_malloc_host": (_i32, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "gq_free_host": (_i32, [_vp]),
    "gq_memcpy": (_i32, [_vp, _vp, C.c_size_t, _vp]),
    "gq_memset": (_i32, [_vp, _i32, C.c_size_t, _vp]),
    "gq_stream_sync": (_i32, [_vp]),
    "gq_kdraws_bytes": (C.c_size_t, [C.POINTER(GqKdraws)]),
    "gq_norm_kdraws": (_i32, [_pp, _u32, _u32, _u64, _u32, _u32, _vp, _vp, _vp, _vp, C.POINTER(GqKdraws), _vp]),
    "gq_reduce_lanes_kdraws": (_i32, [_pp, _u32, _u64, _u64, _u64, _u32, _u32, _u32, _u32, _u64, _u64,
                                      _vp, _vp, _vp, _vp, _f32, _vp, C.POINTER(GqKdraws), _vp]),
    "gq_graph_mean_inproc": (_i32, [_pp, _u32, _u64, C.POINTER(GqConfig), _vp, _pp, _vp, _vp, _vp, _f32, _vp,
                                    _vp, _vp, _vp, _vp, C.POINTER(C.c_void_p)]),
    "gq_graph_launch": (_i32, [_vp, _vp]),
    "gq_graph_destroy": (_i32, [_vp]),
    "gq_quantize_scatter": (_i32, [_vp, _u32, _u32, _u64, _vp, _u32, _u32, _u32, _u32, _u64, _u64, _pp, _u32,
                                   _u64, _vp, _vp]),
    "gq_reduce_slice_multicast": (_i32, [_pp, _u32, _u64, _u64, _u64, _u32, _u32, _u32, _u32, _u64, _u64, _pp,
                                         _u32, _vp, _vp]),
    "gq_p2p_signal": (_i32, [_pp, _u32, _u32, _vp]),
    "gq_p2p_wait": (_i32, [_vp, _u32, _u32, _vp, _vp]),
    "gq_comm_handle_bytes": (C.c_size_t, []),
    "gq_comm_init": (_i32, [_u32, _u32, C.POINTER(GqConfig), _u64, C.POINTER(C.c_void_p)]),
    "gq_comm_handle": (_i32, [_vp, _vp]),
    "gq_comm_connect": (_i32, [_vp, _vp]),
    "gq_comm_info_get": (_i32, [_vp, C.POINTER(GqCommInfo)]),
    "gq_comm_destroy": (_i32, [_vp]),
    "gq_norm_exchange": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "gq_comm_norm": (_i32, [_vp, _pp, _u32, _u64, _vp, _vp, _vp]),
    "gq_comm_quantize": (_i32, [_vp, _pp, _u32, _vp, _u64, _vp, _vp]),
    "gq_allreduce_lanes": (_i32, [_vp, _pp, _u64, _vp, _vp, _vp]),
    "gq_comm_summed": (_vp, [_vp]),
    "gq_comm_mean": (_i32, [_vp, _pp, _u32, _u64, _vp, _vp, _vp, _f32, _vp, _vp, _vp]),
    "gq_sync": (_i32, [_vp, _vp, _vp]),
    "gq_comm_graph": (_i32, [_vp, _pp, _u32, _vp, _vp, _vp, _f32, _vp, _u64, _vp, C.POINTER(C.c_void_p)]),
    "gq_ipc_handle_bytes": (C.c_size_t, []),
    "gq_ipc_get": (_i32, [_vp, _vp]),
    "gq_ipc_open": (_i32, [_vp, C.POINTER(C.c_void_p)]),
    "gq_ipc_close": (_i32, [_vp]),
    "gq_dequant": (_i32, [_vp, _u64, _u64, _vp, _u32, _u32, _u32, _u32, _vp, _vp, _f32, _vp, _vp]),
    "gq_mean_inproc": (_i32, [_pp, _u32, _u64, C.POINTER(GqConfig), _u64, _pp, _vp, _vp, _vp,
                              _f32, _vp, _vp, _vp, _vp, _vp]),
    "gq_baseline_mean_inproc": (_i32, [_pp, _u32, _u64, _u32, _vp, _vp]),
    "gq_check": (_i32, [_vp, _vp]),
}

_lib: C.CDLL | None = None


class GqError(Exception):
    """Base class; subclasses mirror the reference's exception classes."""


class InvalidArgument(GqError, ValueError):
    """std::invalid_argument"""


class LaneOverflow(GqError, OverflowError):
    """std::overflow_error"""


class DomainError(GqError, ValueError):
    """std::domain_error"""


class RuntimeFailure(GqError, RuntimeError):
    """std::runtime_error / CUDA errors"""


_EXC = {GQ_ERR_INVALID: InvalidArgument, GQ_ERR_OVERFLOW: LaneOverflow,
        GQ_ERR_DOMAIN: DomainError, GQ_ERR_RUNTIME: RuntimeFailure, GQ_ERR_CUDA: RuntimeFailure}


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeFailure(
                f"{LIB_PATH} is missing: the sm_100a library must be built "
                "(python -m paper_2305_18627_b200.build); there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.gq_abi_version() != 1:
            raise RuntimeFailure("libgq_b200.so ABI version mismatch")
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != GQ_OK:
        msg = lib().gq_last_error().decode()
        raise _EXC.get(rc, RuntimeFailure)(msg)


def ptr_array(ptrs) -> C.Array:
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
