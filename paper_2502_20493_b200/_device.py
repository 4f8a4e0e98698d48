"""Device plumbing: torch owns device memory and streams; the CUDA library computes."""

from __future__ import annotations

import numpy as np

from . import _lib


def torch():
    import torch as _torch
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("segb200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return t


def stream_ptr(device=None) -> int:
    t = torch()
    return t.cuda.current_stream(device).cuda_stream


def dtype_id(dt) -> int:
    """numpy or torch dtype -> segb dtype id."""
    t = torch()
    if dt in (np.float32, np.dtype(np.float32), t.float32):
        return _lib.F32
    if dt in (np.float64, np.dtype(np.float64), t.float64):
        return _lib.F64
    if dt == t.bfloat16:
        return _lib.BF16
    raise ValueError(f"unsupported dtype {dt}")


def torch_dtype(dt_id: int):
    t = torch()
    return {_lib.F32: t.float32, _lib.F64: t.float64, _lib.BF16: t.bfloat16}[dt_id]


def np_dtype(dt_id: int):
    return {_lib.F32: np.float32, _lib.F64: np.float64}[dt_id]


def to_device(arr: np.ndarray, device=None):
    """Upload a host numpy array (contiguous) to the current CUDA device."""
    t = require_cuda()
    return t.from_numpy(np.ascontiguousarray(arr)).to(device or t.cuda.current_device())
