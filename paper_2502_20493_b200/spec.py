"""Shape algebra of the stride-2 transpose convolution (host side).

Mirrors /root/reference/pkg/src/segconv/engines.py:58-96 (TransposeConvSpec,
output_dims), segregation.py:45-58,91-96 (EffectivePadding, subkernel_dims,
effective_padding) and analysis.py:46-57 (mult_count_segregated). The
arithmetic is done by the C ABI (segb_output_dims & co.), so the host mirror
and the CUDA library share one definition.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from .errors import SpecError


@dataclass(frozen=True)
class EffectivePadding:
    """Input padding for the segregated engine plus the odd-padding swap flag."""

    pad: int
    swap: bool


def effective_padding(pad: int) -> EffectivePadding:
    """segregation.py:91-96: P becomes floor(P/2), with a swap when P is odd."""
    a, b = ctypes.c_int(), ctypes.c_int()
    _lib.check(_lib.lib().segb_effective_padding(int(pad), ctypes.byref(a), ctypes.byref(b)))
    return EffectivePadding(pad=a.value, swap=bool(b.value))


def subkernel_dims(size: int, row_parity: int, col_parity: int) -> tuple[int, int]:
    """segregation.py:53-58: (rows, cols) of sub-kernel (r, s) for side `size`."""
    a, b = ctypes.c_int(), ctypes.c_int()
    _lib.check(_lib.lib().segb_subkernel_dims(int(size), int(row_parity), int(col_parity),
                                              ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


@dataclass(frozen=True)
class TransposeConvSpec:
    """Shape parameters of one stride-2 transpose-convolution layer (engines.py:58-90)."""

    in_h: int
    in_w: int
    kernel_n: int
    pad: int
    c_in: int = 1
    c_out: int = 1
    stride: int = 2

    def __post_init__(self):
        if self.stride != 2:
            raise SpecError(f"stride is fixed at 2, got {self.stride}")
        if self.c_in < 1 or self.c_out < 1:
            raise SpecError(f"channel counts must be >= 1, got {self.c_in}->{self.c_out}")
        _spec_dims(self.in_h, self.in_w, self.kernel_n, self.pad)

    def effective_padding(self) -> EffectivePadding:
        return effective_padding(self.pad)


def _spec_dims(in_h: int, in_w: int, kernel_n: int, pad: int) -> tuple[int, int]:
    a, b = ctypes.c_int(), ctypes.c_int()
    _lib.check(_lib.lib().segb_output_dims(int(in_h), int(in_w), int(kernel_n), int(pad),
                                           ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def output_dims(spec: TransposeConvSpec) -> tuple[int, int]:
    """engines.py:93-96: (2*in_h + 2*pad - n, 2*in_w + 2*pad - n)."""
    return _spec_dims(spec.in_h, spec.in_w, spec.kernel_n, spec.pad)


def mult_count_segregated(spec: TransposeConvSpec) -> int:
    """analysis.py:46-57: live multiplications of one sample (the useful-MAC count)."""
    v = _lib.lib().segb_mult_count_segregated(spec.in_h, spec.in_w, spec.kernel_n, spec.pad,
                                              spec.c_in, spec.c_out)
    if v < 0:
        _lib.check(_lib.SEGB_ERR_SPEC)
    return int(v)


def mult_count_reference(spec: TransposeConvSpec) -> int:
    """analysis.py:40-43: multiplications of the reference engine (Alg. 1), M_h*M_w*n^2*c_in*c_out."""
    oh, ow = output_dims(spec)
    return oh * ow * spec.kernel_n ** 2 * spec.c_in * spec.c_out


def algorithmic_bytes(spec: TransposeConvSpec, batch: int, x_bytes: int, y_bytes: int,
                      w_bytes: int) -> int:
    """in + out + weights, each touched once (no upsampled or padded buffer)."""
    oh, ow = output_dims(spec)
    return (batch * spec.c_in * spec.in_h * spec.in_w * x_bytes
            + batch * spec.c_out * oh * ow * y_bytes
            + spec.c_in * spec.c_out * spec.kernel_n ** 2 * w_bytes)


SAVINGS_UPSAMPLED_TOTAL = "upsampled_total"
SAVINGS_UPSAMPLED_MINUS_INPUT = "upsampled_minus_input"


def memory_savings_bytes(in_h: int, in_w: int, pad: int, c_in: int,
                         mode: str = SAVINGS_UPSAMPLED_TOTAL, element_bytes: int = 4) -> int:
    """analysis.py:60-82: bytes of the bed-of-nails upsampled (and padded) buffer the segregated
    engine never allocates, per sample -- the paper's memory-savings figure. mode
    "upsampled_minus_input" nets out the floor(P/2)-padded raw input buffer."""
    if in_h < 1 or in_w < 1 or c_in < 1:
        raise SpecError(f"dims must be >= 1, got {in_h}x{in_w} with {c_in} channels")
    if pad < 0:
        raise SpecError(f"padding must be >= 0, got {pad}")
    if element_bytes < 1:
        raise SpecError(f"element size must be >= 1 byte, got {element_bytes}")
    upsampled = (2 * in_h - 1 + 2 * pad) * (2 * in_w - 1 + 2 * pad) * c_in * element_bytes
    if mode == SAVINGS_UPSAMPLED_TOTAL:
        return upsampled
    if mode == SAVINGS_UPSAMPLED_MINUS_INPUT:
        eff = pad // 2
        return upsampled - (in_h + 2 * eff) * (in_w + 2 * eff) * c_in * element_bytes
    raise ValueError(f"unknown savings mode {mode!r}, expected one of "
                     f"{(SAVINGS_UPSAMPLED_TOTAL, SAVINGS_UPSAMPLED_MINUS_INPUT)}")
