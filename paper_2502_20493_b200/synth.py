"""Synthetic inputs generated on the device with the reference's exact bits.

synth.py:20-56 of the reference: element i = float32(float64(splitmix64(seed + i))
* 2**-64). The batched stream (B, C, H, W) = unit_floats(B*C*H*W, seed) makes
sample j equal to gen_synthetic(C, H, W, seed + j*C*H*W), so any
sample of a multi-GB device batch is reproducible by the per-sample oracle.
"""

from __future__ import annotations

from . import _device, _lib

_MASK = (1 << 64) - 1


def splitmix64(value: int) -> int:
    """Host copy of the stateless splitmix64 output function (seed derivation only)."""
    z = (value + 0x9E3779B97F4A7C15) & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def harness_seeds(seed: int, index: int) -> tuple[int, int]:
    """bench.py:299-300 of the reference: per-layer input and bank seeds."""
    input_seed = splitmix64((seed & _MASK) + 2 * index)
    return input_seed, splitmix64(input_seed + 1)


def device_unit_floats(shape, seed: int, dtype=None, device=None):
    """torch tensor of `shape` on the GPU filled by the segb_unit_floats kernel."""
    t = _device.require_cuda()
    dtype = dtype or t.float32
    out = t.empty(shape, dtype=dtype, device=device or t.cuda.current_device())
    _lib.check(_lib.lib().segb_unit_floats(out.data_ptr(), _device.dtype_id(dtype), out.numel(),
                                           seed & _MASK, _device.stream_ptr(out.device)))
    return out
