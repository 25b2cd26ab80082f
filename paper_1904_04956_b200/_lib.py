"""ctypes binding of libds.so (the C ABI declared in include/ds_blstm.h).

ctypes releases the GIL around every foreign call, so learner threads can
issue GPU work concurrently.  There is no fallback: if the shared object is
missing or fails to load, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libds.so")

DS_OK = 0
DS_ERR_ARG = -1
DS_ERR_CUDA = -2
DS_ERR_NONFINITE = -3
DS_PREC_BF16 = 0
DS_PREC_FP32 = 1

# Every symbol of include/ds_blstm.h with its ctypes signature.
_VP = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F32 = ctypes.c_float
SIGNATURES = {
    "ds_blstm_param_dim": (_I64, [_VP]),
    "ds_blstm_create": (_I32, [_VP, _I32, ctypes.POINTER(_VP)]),
    "ds_blstm_destroy": (_I32, [_VP]),
    "ds_blstm_set_dataset": (_I32, [_VP, _VP, _VP, _I64]),
    "ds_blstm_cast_snapshot": (_I32, [_VP, _VP, _VP]),
    "ds_blstm_fwd_bwd": (_I32, [_VP, _VP, _I32, _VP, _VP, _VP, _VP]),
    "ds_blstm_loss": (_I32, [_VP, _VP, _I32, _VP, _VP, _VP]),
    "ds_blstm_train_step": (_I32, [_VP, _VP, _I32, _VP, _VP, _VP, _F32, _F32, _VP, _VP, _VP]),
    "ds_sgd_momentum": (_I32, [_VP, _VP, _VP, _F32, _F32, _I64, _VP, _VP, _VP]),
    "ds_adpsgd_mix": (_I32, [_VP, _VP, _I64, _VP]),
    "ds_group_reduce": (_I32, [_I32, _I32, _VP, _VP, _VP, _VP, _I64, _I32, _F32, _F32, _I32, _F32, _VP]),
    "ds_average": (_I32, [_I32, _VP, _VP, _I64, _VP]),
    "ds_blstm_set_grad_scale": (_I32, [_VP, _F32]),
    "ds_blstm_set_profile": (_I32, [_VP, _I32]),
    "ds_blstm_read_loss": (_I32, [_VP, _VP, _VP, ctypes.POINTER(ctypes.c_float)]),
    "ds_blstm_profile_read": (_I32, [_VP, _VP, _I32]),
    "ds_blstm_kernel_count": (_I32, [_VP]),
    "ds_blstm_profile_list": (_I32, [_VP, _VP, _VP, _I32, _VP]),
    "ds_debug_gemm_trace": (_I32, [_VP, _I32]),
    "ds_debug_bptt_trace": (_I32, [_VP, _I32]),
    "ds_debug_gemm_bf16": (_I32, [_VP, _I64, _I32, _VP, _I64, _I32, _VP, _I64, _I32, _I32, _I32, _VP]),
    "ds_debug_lstm_fwd": (_I32, [_I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ds_debug_lstm_bwd": (_I32, [_I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ds_ipc_export": (_I32, [_VP, _VP, ctypes.POINTER(_I64)]),
    "ds_ipc_open": (_I32, [_VP, _I64, ctypes.POINTER(_VP), ctypes.POINTER(_VP)]),
    "ds_ipc_close": (_I32, [_VP]),
    "ds_device_copy": (_I32, [_VP, _VP, _I64, _VP]),
    "ds_enable_peer_access": (_I32, [_I32, _I32]),
    "ds_blstm_snapshot_ptr": (_VP, [_VP]),
    "ds_blstm_snapshot_aux": (_I32, [_VP, _VP, _VP]),
    "ds_peer_barrier": (_I32, [_I32, _VP, _VP, _I32, _VP, _VP, _VP, ctypes.c_double, _VP]),
    "ds_peer_lock": (_I32, [_VP, ctypes.c_uint32, _VP, ctypes.c_double, _VP]),
    "ds_peer_unlock": (_I32, [_VP, _VP]),
    "ds_update_mix": (_I32, [_VP, _VP, _VP, _VP, _VP, _F32, _F32, _I64, _VP, _VP]),
    "ds_digest": (_I32, [_VP, _I64, _VP, _VP]),
    "ds_shard_step_range": (_I32, [_I32, _I32, _VP, _VP, _VP, _VP, _I64, _I32, _F32, _F32, _I32, _F32, _I64, _I64,
                                   _I32, _VP]),
    "ds_shard_step": (_I32, [_I32, _I32, _VP, _VP, _VP, _VP, _I64, _I32, _F32, _F32, _I32, _F32, _VP]),
    "ds_pair_mix": (_I32, [_VP, _VP, _VP, _VP, _I64, _I32, _VP]),
    "ds_blstm_set_precision": (_I32, [_VP, _I32]),
    "ds_blstm_get_precision": (_I32, [_VP]),
    "ds_debug_gemm_tf32x3": (_I32, [_VP, _I64, _VP, _I64, _VP, _I64, _I32, _I32, _I32, _I32, _VP]),
    "ds_blstm_set_group": (_I32, [_VP, _VP]),
    "ds_last_error": (ctypes.c_char_p, []),
}


class DsError(RuntimeError):
    """CUDA-level failure inside libds."""


class DsCfg(ctypes.Structure):
    _fields_ = [
        ("layers", _I32),
        ("input_dim", _I32),
        ("bottleneck", _I32),
        ("classes", _I32),
        ("frames", _I32),
        ("max_batch", _I32),
    ]


DS_MAX_GROUP = 16


class DsGroupDesc(ctypes.Structure):
    """ds_group_desc of include/ds_blstm.h (fused SSGD group step)."""

    _fields_ = [
        ("n", _I32), ("me", _I32), ("my_rank", _I32), ("nchunks", _I32), ("divisor", _F32), ("max_blocks", _I32),
        ("ranks", _I32 * DS_MAX_GROUP),
        ("thetas", _VP * DS_MAX_GROUP), ("grads", _VP * DS_MAX_GROUP), ("snaps", _VP * DS_MAX_GROUP),
        ("flags", _VP * DS_MAX_GROUP),
        ("own_flags", _VP), ("pair_epochs", _VP), ("err", _VP), ("timeout_s", ctypes.c_double),
    ]


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libds.so (building nothing: run `make -C paper_1904_04956_b200/csrc`
    or __graft_entry__.build() first)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DsError(f"libds.so not built: {LIB_PATH} is missing (run __graft_entry__.build())")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    return load().ds_last_error().decode(errors="replace")


def check(rc: int, what: str = "libds") -> None:
    """Map a C return code onto the reference's exception types
    (ValueError for shape/config/non-finite, objectives.py:186-191,261-262)."""
    if rc == DS_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc in (DS_ERR_ARG, DS_ERR_NONFINITE):
        raise ValueError(msg)
    raise DsError(msg)


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
