"""Parity segregation of square kernels -- on the device (K1).

Mirrors /root/reference/pkg/src/segconv/segregation.py: SubKernelSet
(:23-42), segregate_kernel (:61-70), merge_subkernels (:73-88). The split and
its inverse are bit-exact permutations run by the segb_segregate /
segb_merge kernels; the host only validates shapes (same ShapeError texts as
the reference) and moves arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .errors import ShapeError
from .spec import EffectivePadding, effective_padding, subkernel_dims  # noqa: F401 (re-export)


@dataclass(frozen=True)
class SubKernelSet:
    """The four parity sub-kernels of one square kernel of side `size` (segregation.py:23-42)."""

    size: int
    k00: np.ndarray
    k01: np.ndarray
    k10: np.ndarray
    k11: np.ndarray

    def sub(self, row_parity: int, col_parity: int) -> np.ndarray:
        return (self.k00, self.k01, self.k10, self.k11)[2 * row_parity + col_parity]

    def element_count(self) -> int:
        return self.k00.size + self.k01.size + self.k10.size + self.k11.size


def require_square_kernel(arr) -> np.ndarray:
    """tensors.py:63-73: 2-D, square, side >= 2, float."""
    if not isinstance(arr, np.ndarray):
        arr = np.asarray(arr, dtype=np.float32)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise ShapeError(f"kernel must be square, got shape {arr.shape}")
    if arr.shape[0] < 2:
        raise ShapeError(f"kernel side must be >= 2, got {arr.shape[0]}")
    if not np.issubdtype(arr.dtype, np.floating):
        raise ShapeError(f"kernel must hold floats, got dtype {arr.dtype}")
    return arr


def _block_sizes(n: int):
    return [subkernel_dims(n, r, s) for r in (0, 1) for s in (0, 1)]


def _device_permute(src: np.ndarray, n: int, count: int, merge: bool) -> np.ndarray:
    t = _device.require_cuda()
    dt = src.dtype
    if dt not in (np.float32, np.float64):
        work = src.astype(np.float64)
    else:
        work = src
    d_src = _device.to_device(work.reshape(-1))
    d_dst = t.empty_like(d_src)
    fn = _lib.lib().segb_merge if merge else _lib.lib().segb_segregate
    _lib.check(fn(d_src.data_ptr(), _device.dtype_id(work.dtype), count, n, d_dst.data_ptr(),
                  _device.stream_ptr()))
    return d_dst.cpu().numpy().astype(dt, copy=False)


def segregate_kernel(kernel) -> SubKernelSet:
    """Split a square kernel (side >= 2) into its four parity sub-kernels (K1 on device)."""
    k = require_square_kernel(kernel)
    n = k.shape[0]
    flat = _device_permute(np.ascontiguousarray(k), n, 1, merge=False)
    subs, off = [], 0
    for rows, cols in _block_sizes(n):
        subs.append(flat[off:off + rows * cols].reshape(rows, cols).copy())
        off += rows * cols
    return SubKernelSet(size=n, k00=subs[0], k01=subs[1], k10=subs[2], k11=subs[3])


def merge_subkernels(subs: SubKernelSet) -> np.ndarray:
    """Reassemble the original kernel; exact inverse of segregate_kernel (K1 merge on device)."""
    n = subs.size
    for r in (0, 1):
        for s in (0, 1):
            expected = subkernel_dims(n, r, s)
            actual = subs.sub(r, s).shape
            if tuple(actual) != expected:
                raise ShapeError(f"sub-kernel ({r},{s}) has shape {actual}, "
                                 f"expected {expected} for size {n}")
    dt = np.result_type(subs.k00, subs.k01, subs.k10, subs.k11)
    packed = np.concatenate([np.asarray(subs.sub(r, s), dtype=dt).reshape(-1)
                             for r in (0, 1) for s in (0, 1)])
    return _device_permute(packed, n, 1, merge=True).reshape(n, n)
