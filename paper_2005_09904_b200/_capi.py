"""ctypes binding of include/bqg_capi.h (libbiqgemm_b200.so).

This is the same binding a Python caller of the reference's C++ API would
add.  Loading fails loudly when the library has not been
built: there is no Python or CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# BQG_LIB_VARIANT selects an experimental build under lib/ (tuning runs only).
_LIB_PATH = Path(__file__).resolve().parent / "lib" / (
    f"libbiqgemm_b200.{os.environ['BQG_LIB_VARIANT']}.so" if os.environ.get("BQG_LIB_VARIANT") else "libbiqgemm_b200.so")

BQG_OK = 0
BQG_ERR_INVALID_ARGUMENT = 1
BQG_ERR_CUDA = 2
BQG_ERR_NO_DEVICE = 3
BQG_ERR_OUT_OF_MEMORY = 4
BQG_ERR_FORMAT = 5
BQG_ERR_BAD_MAGIC = 6
BQG_ERR_BAD_VERSION = 7
BQG_ERR_TRUNCATED = 8
BQG_ERR_RANGE = 9
BQG_ERR_IO = 10
BQG_ERR_WORKSPACE = 11
BQG_ERR_COMM = 12

LUT_TABLE_MAJOR = 0
LUT_KEY_MAJOR = 1
LUT_DP = 0
LUT_NAIVE = 1
FORWARD_FAST = 0
FORWARD_EXACT = 1
FORWARD_EXACT_NAIVE = 2

sz = C.c_size_t
u32 = C.c_uint
u64 = C.c_uint64
vp = C.c_void_p
i32 = C.c_int
f32 = C.c_float
f64 = C.c_double
P = C.POINTER


class KernelStats(C.Structure):
    """bqg_kernel_stats == OpCounters + KernelStats (kernel.hpp:23-46)."""

    _fields_ = [
        ("lut_build_ops", u64),
        ("lookups", u64),
        ("accumulate_ops", u64),
        ("fma_ops", u64),
        ("build_seconds", f64),
        ("query_seconds", f64),
        ("replace_seconds", f64),
    ]


BcastFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)
AllGatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class Collectives(C.Structure):
    """bqg_collectives: the broadcast / all-gather the sharded call uses."""

    _fields_ = [("ctx", C.c_void_p), ("broadcast", BcastFn), ("allgather", AllGatherFn)]


class Call(C.Structure):
    """bqg_call: one entry of a grouped biqgemm launch."""

    _fields_ = [("d_keys_tiled", vp), ("d_alpha", vp), ("d_x", vp), ("d_y", vp)]


class ShardCall(C.Structure):
    """bqg_shard_call: one entry of a grouped row-sharded launch (this rank's shard)."""

    _fields_ = [("d_keys_tiled_shard", vp), ("d_alpha_shard", vp)]


# name -> (restype, argtypes).  Every symbol declared in include/bqg_capi.h.
SIGNATURES = {
    "bqg_status_string": (C.c_char_p, [i32]),
    "bqg_last_error_message": (C.c_char_p, []),
    "bqg_abi_version": (i32, []),
    "bqg_random_uniform_f32": (i32, [vp, sz, sz, u64, f32, f32]),
    "bqg_random_normal_f32": (i32, [vp, sz, sz, u64]),
    "bqg_random_uniform_f64": (i32, [vp, sz, sz, u64, f64, f64]),
    "bqg_random_normal_f64": (i32, [vp, sz, sz, u64]),
    "bqg_plan_tiles": (i32, [sz, sz, sz, u32, sz, sz, P(sz), P(sz)]),
    "bqg_footprint": (i32, [u64, u64, u32, u64, u32, u32, P(u64)]),
    "bqg_op_counters": (i32, [sz, sz, sz, u32, u32, i32, P(u64)]),
    "bqg_tiled_key_bytes": (sz, [sz, sz, u32, u32]),
    "bqg_bqgm_parse": (i32, [vp, sz, P(sz), P(sz), P(u32), P(u32), vp, vp]),
    "bqg_bqgm_serialize": (i32, [vp, vp, sz, sz, u32, u32, vp, P(sz)]),
    "bqg_quantize_greedy_f32": (i32, [vp, sz, sz, u32, vp, vp, vp]),
    "bqg_quantize_greedy_f64": (i32, [vp, sz, sz, u32, vp, vp, vp]),
    "bqg_pack_keys": (i32, [vp, sz, sz, u32, vp, vp]),
    "bqg_tile_keys": (i32, [vp, sz, sz, u32, u32, vp, vp]),
    "bqg_build_lut_f32": (i32, [vp, sz, sz, u32, sz, sz, i32, i32, vp, P(u64), vp]),
    "bqg_build_lut_f64": (i32, [vp, sz, sz, u32, sz, sz, i32, i32, vp, P(u64), vp]),
    "bqg_build_lut_f64x": (i32, [vp, sz, sz, u32, sz, sz, i32, i32, vp, P(u64), vp]),
    "bqg_biqgemm_workspace_bytes": (sz, [sz, sz, sz, u32, u32]),
    "bqg_biqgemm_f32": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, u32, vp, sz, i32, vp]),
    "bqg_biqgemm_grouped_workspace_bytes": (sz, [sz, sz, sz, u32, u32, sz]),
    "bqg_biqgemm_form": (i32, [sz, sz, sz, u32, u32]),
    "bqg_gemm_unpack_f32": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, vp]),
    "bqg_bandwidth_probe": (i32, [vp, sz, sz, vp, sz, vp, i32, vp]),
    "bqg_biqgemm_grouped_f32": (i32, [vp, sz, sz, sz, sz, sz, u32, u32, vp, sz, i32, vp]),
    "bqg_layers_forward_host": (i32, [vp, sz, vp, sz, sz, vp, i32, vp]),
    "bqg_biqgemm_exact_workspace_bytes": (sz, [sz, sz, sz, u32, u32]),
    "bqg_biqgemm_exact_f32": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, u32, vp, sz, vp]),
    "bqg_biqgemm_exact_f64": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, u32, vp, sz, vp]),
    "bqg_biqgemm_exact_ex_f32": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, u32, i32, vp, sz, P(KernelStats), vp]),
    "bqg_biqgemm_exact_ex_f64": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, u32, i32, vp, sz, P(KernelStats), vp]),
    "bqg_layer_create_from_weights": (i32, [vp, sz, sz, u32, u32, P(vp)]),
    "bqg_layer_create_from_device_weights": (i32, [vp, sz, sz, u32, u32, P(vp)]),
    "bqg_layer_create_from_keys": (i32, [vp, vp, sz, sz, u32, u32, P(vp)]),
    "bqg_layer_load_bqgm": (i32, [vp, sz, P(vp)]),
    "bqg_layer_destroy": (None, [vp]),
    "bqg_layer_shape": (i32, [vp, P(sz), P(sz), P(u32), P(u32)]),
    "bqg_layer_export": (i32, [vp, vp, vp, vp]),
    "bqg_layer_device_tiled_keys": (vp, [vp]),
    "bqg_layer_device_keys": (vp, [vp]),
    "bqg_layer_device_alpha": (vp, [vp]),
    "bqg_layer_forward_host": (i32, [vp, vp, sz, sz, vp, i32, P(KernelStats)]),
    "bqg_layer_forward_device": (i32, [vp, vp, sz, sz, vp, i32, i32, vp]),
    "bqg_shard_rows": (i32, [sz, i32, i32, P(sz), P(sz), P(sz)]),
    "bqg_nccl_available": (i32, []),
    "bqg_nccl_unique_id": (i32, [vp]),
    "bqg_nccl_comm_init": (i32, [vp, i32, i32, P(vp)]),
    "bqg_nccl_comm_destroy": (i32, [vp]),
    "bqg_nccl_collectives": (i32, [vp, P(Collectives)]),
    "bqg_biqgemm_sharded_workspace_bytes": (sz, [sz, sz, sz, u32, u32, i32]),
    "bqg_biqgemm_sharded_f32": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, u32, i32, i32, P(Collectives), vp, sz,
                                      vp]),
    "bqg_biqgemm_grouped_sharded_workspace_bytes": (sz, [sz, sz, sz, u32, u32, sz, i32]),
    "bqg_biqgemm_grouped_sharded_p2p_workspace_bytes": (sz, [sz, sz, sz, u32, u32, sz, i32]),
    "bqg_biqgemm_grouped_sharded_p2p_f32": (i32, [vp, sz, vp, sz, vp, sz, sz, sz, u32, u32, i32, i32, P(Collectives),
                                                  vp, sz, i32, vp]),
    "bqg_biqgemm_sharded_p2p_workspace_bytes": (sz, [sz, sz, sz, u32, u32, i32]),
    "bqg_biqgemm_sharded_p2p_f32": (i32, [vp, vp, vp, sz, vp, sz, sz, sz, u32, u32, i32, i32, P(Collectives), vp,
                                          sz, vp]),
    "bqg_rekey_mu8_columns": (sz, [sz, u32]),
    "bqg_rekey_mu8": (i32, [vp, sz, sz, u32, u32, vp, vp]),
    "bqg_layer_fast_shape": (i32, [vp, P(sz), P(u32)]),
    "bqg_ipc_get_handle": (i32, [vp, vp, P(sz)]),
    "bqg_ipc_open_handle": (i32, [vp, sz, P(vp)]),
    "bqg_ipc_close_handle": (i32, [vp]),
    "bqg_biqgemm_grouped_sharded_f32": (i32, [vp, sz, vp, sz, vp, sz, sz, sz, u32, u32, i32, i32, P(Collectives), vp,
                                              sz, i32, vp]),
}


class BiqgemmError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status


class InvalidArgument(BiqgemmError, ValueError):
    """std::invalid_argument in the reference."""


class FormatError(BiqgemmError):
    """biqgemm::FormatError (model_io.hpp:14)."""


class BadMagicError(FormatError):
    pass


class BadVersionError(FormatError):
    pass


class TruncatedError(FormatError):
    pass


class RangeError(FormatError):
    pass


class NoDeviceError(BiqgemmError):
    pass


_EXC = {
    BQG_ERR_INVALID_ARGUMENT: InvalidArgument,
    BQG_ERR_FORMAT: FormatError,
    BQG_ERR_BAD_MAGIC: BadMagicError,
    BQG_ERR_BAD_VERSION: BadVersionError,
    BQG_ERR_TRUNCATED: TruncatedError,
    BQG_ERR_RANGE: RangeError,
    BQG_ERR_NO_DEVICE: NoDeviceError,
}


def _load() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_2005_09904_b200.build` "
            "(there is no fallback implementation)"
        )
    lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
LIB_PATH = str(_LIB_PATH)


def check(status: int) -> None:
    if status != BQG_OK:
        msg = lib.bqg_last_error_message().decode(errors="replace")
        raise _EXC.get(status, BiqgemmError)(status, msg)
