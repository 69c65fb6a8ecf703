"""ctypes binding of ``libscadles_b200.so`` (the C-ABI in ``include/scadles_b200.h``).

There is no fallback: if the library is missing or no CUDA device is present, every compute
entry point raises.  Status codes map to the reference's exception types: invalid arguments
raise ``ValueError`` (as ``streamsgd.comm`` does), everything else ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint8, c_uint32, c_void_p
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libscadles_b200.so"
if os.environ.get("SG_LIB_PATH"):  # diagnostic builds only (tools/checked_run.py, tools/stamps.py)
    LIB_PATH = Path(os.environ["SG_LIB_PATH"])

SG_OK = 0
SG_ERR_INVALID = -1
SG_ERR_CUDA = -2
SG_ERR_WORKSPACE = -3
SG_ERR_UNSUPPORTED = -4


class GateStateC(ctypes.Structure):
    """sg_gate_state (64 bytes), the device mirror of comm.CompressionState."""

    _fields_ = [
        ("cr", c_double),
        ("delta", c_double),
        ("ewma_factor", c_double),
        ("ewma_full", c_double),
        ("ewma_topk", c_double),
        ("n_compressed", c_int64),
        ("n_uncompressed", c_int64),
        ("raw_gate", c_int32),
        ("initialized", c_int32),
    ]


GATE_STATE_DTYPE = np.dtype(
    [
        ("cr", "<f8"),
        ("delta", "<f8"),
        ("ewma_factor", "<f8"),
        ("ewma_full", "<f8"),
        ("ewma_topk", "<f8"),
        ("n_compressed", "<i8"),
        ("n_uncompressed", "<i8"),
        ("raw_gate", "<i4"),
        ("initialized", "<i4"),
    ]
)
assert GATE_STATE_DTYPE.itemsize == ctypes.sizeof(GateStateC) == 64

# name -> (restype, argtypes); every symbol include/scadles_b200.h declares.
_P = c_void_p
SIGNATURES = {
    "sg_abi_version": (c_int, []),
    "sg_status_string": (c_char_p, [c_int]),
    "sg_topk_count": (c_int64, [c_int64, c_double]),
    "sg_topk_workspace_bytes_f32": (c_size_t, [c_int, c_int64, c_int64]),
    "sg_topk_workspace_bytes_f64": (c_size_t, [c_int, c_int64, c_int64]),
    "sg_topk_workspace_zero_bytes_f32": (c_size_t, [c_int, c_int64, c_int64]),
    "sg_topk_workspace_bytes_fused_f32": (c_size_t, [c_int, c_int64, c_int64]),
    "sg_topk_workspace_zero_bytes_fused_f32": (c_size_t, [c_int, c_int64, c_int64]),
    "sg_topk_gate_fused_f32": (c_int, [_P, c_int, c_int64, c_int64, c_int64, _P, _P, _P, _P, _P, _P, _P, _P, c_size_t, _P]),
    "sg_topk_stats_fused_f32": (c_int, [c_int, c_int64, c_int64, _P, c_size_t, _P, _P]),
    "sg_topk_gate_f32": (c_int, [_P, c_int, c_int64, c_int64, c_int64, _P, _P, _P, _P, _P, _P, _P, _P, c_size_t, _P]),
    "sg_topk_gate_f64": (c_int, [_P, c_int, c_int64, c_int64, c_int64, _P, _P, _P, _P, _P, _P, _P, c_size_t, _P]),
    "sg_gate_update": (c_int, [_P, c_int, _P, _P, _P, _P]),
    "sg_topk_segments_f32": (c_int, [c_int, c_int64, c_int64]),
    "sg_topk_phases_f32": (c_int, [c_int, c_int64, c_int64, _P, c_size_t, _P, c_int64, _P]),
    "sg_topk_stats_f32": (c_int, [c_int, c_int64, c_int64, _P, c_size_t, _P, _P]),
    "sg_topk_stats_f64": (c_int, [c_int, c_int64, c_int64, _P, c_size_t, _P, _P]),
    "sg_aggregate_workspace_bytes": (c_size_t, [c_int, c_int64]),
    "sg_weighted_aggregate_f32": (
        c_int,
        [c_int, POINTER(c_double), _P, _P, c_int64, _P, _P, _P, _P, c_int64, _P, _P, _P,
         c_double, c_double, c_double, c_int, c_int, _P, c_size_t, _P],
    ),
    "sg_weighted_aggregate_f64": (
        c_int,
        [c_int, POINTER(c_double), _P, _P, c_int64, _P, _P, _P, _P, c_int64, _P, _P, _P,
         c_double, c_double, c_double, c_int, _P, c_size_t, _P],
    ),
    "sg_weighted_aggregate_peers_f32": (
        c_int,
        [c_int, POINTER(c_double), _P, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p), c_int64,
         _P, _P, _P, c_double, c_double, c_double, c_int, c_int, c_int, c_int, _P],
    ),
    "sg_gather_bytes": (c_int, [c_int, POINTER(c_void_p), c_int64, _P, _P]),
    "sg_multicast_copy_u32": (c_int, [_P, _P, c_int64, _P]),
    "sg_peer_signal_wait": (c_int, [c_int, c_int, POINTER(c_void_p), c_int, c_uint32, _P, _P, c_int, POINTER(c_void_p),
                                    c_int64, _P, _P]),
    "sg_weighted_partial_f32": (
        c_int,
        [c_int, POINTER(c_double), _P, _P, c_int64, _P, _P, _P, _P, c_int64, _P, _P, c_int, _P, c_size_t, _P],
    ),
    "sg_peer_slice_len": (c_int64, [c_int64, c_int]),
    "sg_peer_reduce_slice_f32": (
        c_int,
        [c_int, POINTER(c_void_p), POINTER(c_double), c_int, _P, c_int, c_int64, _P, _P],
    ),
    "sg_peer_reduce_push_f32": (
        c_int,
        [c_int, POINTER(c_void_p), POINTER(c_double), c_int, _P, c_int, c_int64, POINTER(c_void_p), _P],
    ),
    "sg_dense_exchange_flag_words": (c_size_t, [c_int64, c_int]),
    "sg_nvls_reduce_bcast_f32": (c_int, [c_int, c_int, _P, _P, c_int64, _P, c_int, _P]),
    "sg_dense_exchange_f32": (
        c_int,
        [c_int, c_int, c_int, POINTER(c_double), _P, c_int64, c_int64, POINTER(c_void_p), POINTER(c_void_p),
         POINTER(c_void_p), c_uint32, _P, c_int, _P, _P, _P, c_double, c_double, c_double, c_int, _P],
    ),
    "sg_peer_allgather_sgd_f32": (
        c_int,
        [c_int, POINTER(c_void_p), c_int, _P, c_int, c_int64, _P, _P, _P, c_double, c_double, c_double, c_int, _P],
    ),
    "sg_sgd_momentum_f32": (c_int, [_P, _P, _P, c_int64, c_double, c_double, c_double, c_int, _P]),
    "sg_sgd_momentum_f64": (c_int, [_P, _P, _P, c_int64, c_double, c_double, c_double, c_int, _P]),
    "sg_gather_batch_f64": (c_int, [_P, _P, _P, c_int64, _P, c_int64, _P, _P, _P]),
    "sg_gather_batch_f32": (c_int, [_P, _P, _P, c_int64, _P, c_int64, _P, _P, _P]),
    "sg_resolve_stream_rows": (c_int, [c_int, _P, _P, _P, _P, _P, c_int64, _P, _P]),
    "sg_inject_rows": (c_int, [c_int, _P, _P, c_int, _P, _P, _P, _P, _P, _P]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2301_08897_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status == SG_OK:
        return
    msg = load().sg_status_string(status).decode()
    if status in (SG_ERR_INVALID,):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (status {status})")


def weights_ptr(weights: np.ndarray):
    w = np.ascontiguousarray(weights, dtype=np.float64)
    return w, w.ctypes.data_as(POINTER(c_double))
