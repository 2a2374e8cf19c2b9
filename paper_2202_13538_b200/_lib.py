"""ctypes binding of the C ABI in include/walkjoin_b200.h.

The CUDA library is built in-tree (``build.py``) and loaded from this
directory.  There is no fallback: if the library or a CUDA device is missing
the calls raise ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# WJ_LIB: an alternative build of the same library (A/B measurements, profiles/ab_variant.py)
LIB_PATH = os.environ.get("WJ_LIB") or os.path.join(_HERE, "_walkjoin_b200.so")

WJ_OK, WJ_ERR_ARG, WJ_ERR_CUDA, WJ_ERR_UNSUPPORTED = 0, 1, 2, 3
DTYPE_CODES = {torch.float32: 0, torch.float64: 1, torch.bfloat16: 2, torch.float16: 3}

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64

# name -> argtypes (all return int status)
SIGNATURES = {
    "wj_sample_walks": [P, ctypes.c_int, P, I64, I64, I64, I32, I32, U64, P, P, P],
    "wj_sample_node_walks": [P, ctypes.c_int, P, I64, I32, I32, U64, P, P, P],
    "wj_sample_walks_typed": [P, ctypes.c_int, P, P, P, I32, P, I32, I64, I64, I64, I32, I32, U64, P, P],
    "wj_typed_csr": [P, ctypes.c_int, P, P, I64, I32, P, P, P],
    "wj_rpe_count": [P, I64, I32, I32, I64, P, P],
    "wj_rpe_fill": [P, I64, I32, I32, I64, P, P, P, P, P, P],
    "wj_intern_insert": [P, P, P, I64, I64, P, P, I64, P, P],
    "wj_intern_assign": [P, I64, P, P, I64, P, P],
    "wj_join": [P, I64, I32, P, P, P, P, P, I32, I32, I32, P, I64, P, P, P, I32, I64, P],
    "wj_join_encode": [P, I64, I32, P, P, P, P, P, P, P, P, I32, I32, I32, P, I64, P, P, I32, ctypes.c_float,
                       U64, P, P, P, P, P],
    "wj_join_cross": [P, I64, I32, P, P, P, I32, P, P],
    "wj_score_shared": [P, I64, P, P, P, P, I32, I32, I32, P, P, P, P, P, P],
    "wj_vindex_count": [P, P, I64, P, I32, I32, P, P],
    "wj_vindex_fill": [P, P, I64, P, I32, I32, P, P, P, P],
    "wj_table_rows_f16": [P, I64, I32, I32, P, P],
    "wj_join_encode_simt": [P, I64, I32, P, P, P, I32, I32, I32, P, I64, P, P, I32, ctypes.c_float, U64,
                            P, P, P, P, P],
    "wj_encoder_tail": [P, P, P, P, I64, I32, I32, P, P, ctypes.c_float, P, P, I32, P, P, P],
    "wj_adam": [P, P, P, P, I32, I32, ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                P, P, P, P],
    "wj_sum_partials": [P, I32, I32, P, P],
    "wj_stepper_create": [P, P, P, P, P, P, P, I32, I32, I32, I32, P, P, P, P, ctypes.c_float, ctypes.c_float, U64,
                          ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, P, P, P, P, P, I32, P, P],
    "wj_stepper_run": [P, P, P, I64, P, I64, P, P],
    "wj_stepper_destroy": [P],
    "wj_stepper_encode": [P, P, I64, P, I64, P],
    "wj_stepper_grads": [P, P, P, I64, P, I64, P, P],
    "wj_stepper_apply": [P, P, P, P],
    "wj_stepper_grads_shard": [P, P, P, I64, P, I64, I64, I64, I32, I32, P, P],
    "wj_stepper_apply_rows": [P, P, I32, P, P],
    "wj_gather_rpe": [P, I64, P, I64, I32, P, I32, P, P],
    "wj_export_dicts": [P, P, P, P, P, I64, I32, I32, P, P, P, P],
    "wj_lookup": [P, P, I64, P, P, P, P, P],
    "wj_surl_pack": [P, I64, I32, P, P, P, P, P, P],
    "wj_surl_unpack": [P, I64, I32, P, P, P, P, P, P],
    "wj_planner_create": [P, I64, I32, P, I64, I64, I32, I32, I32, P, I64, P],
    "wj_upload": [P, P, I64, I32],
    "wj_planner_destroy": [P],
    "wj_planner_set_rng": [P, P],
    "wj_planner_get_rng": [P, P],
    "wj_planner_next": [P, P, P, I64, P, P, P],
    "wj_planner_start_epoch": [P, P, P, P, I32, I64],
    "wj_group_queries": [P, I64, I32, I32, P, P],
    "wj_planner_acquire": [P, P, P, P],
    "wj_planner_release": [P, I32],
    "wj_planner_stop": [P],
    "wj_train_epoch": [P, P, P, P, I32, I64, I32, P, P, I32, P, P, I64, P, P, P, P],
}

_lib = None


def load():
    """Load the in-tree CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA extension {LIB_PATH} is missing; run `python -m paper_2202_13538_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = ctypes.c_int
        lib.wj_last_error.restype = ctypes.c_char_p
        lib.wj_last_error.argtypes = []
        lib.wj_abi_version.restype = ctypes.c_int
        if lib.wj_abi_version() != 1:
            raise RuntimeError("walkjoin_b200 ABI version mismatch")
        _lib = lib
    return _lib


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2202_13538_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device; no CPU fallback")
    return dev


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def sm_count_of(device) -> int:
    return torch.cuda.get_device_properties(device).multi_processor_count


def stream_handle(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != WJ_OK:
        msg = lib.wj_last_error().decode(errors="replace")
        if rc == WJ_ERR_ARG:
            raise ValueError(f"{name}: {msg}")
        if rc == WJ_ERR_UNSUPPORTED:
            raise NotImplementedError(f"{name}: {msg}")
        raise RuntimeError(f"{name}: {msg}")
