"""Host-side tests (no GPU): the C ABI loads and exports every declared symbol,
shape algebra/counts match the reference's golden values, and the drop-in API
raises the reference's exceptions before touching the device."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2502_20493_b200 as P
from paper_2502_20493_b200 import _lib
from tests.conftest import ROOT


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "segb200.h")).read()
    return sorted(set(re.findall(r"\b(segb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES)
    assert _lib.lib().segb_abi_version() == 2


def test_library_has_sm100a_code():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("nh,n,pad,expected", [(4, 3, 0, 5), (4, 5, 2, 7), (4, 4, 2, 8)])
def test_output_dims(nh, n, pad, expected):
    assert P.output_dims(P.TransposeConvSpec(in_h=nh, in_w=nh, kernel_n=n, pad=pad)) == (expected, expected)
    assert P.output_dims(P.TransposeConvSpec(in_h=3, in_w=5, kernel_n=2, pad=0)) == (4, 8)


@pytest.mark.parametrize("kwargs", [
    dict(in_h=1, in_w=1, kernel_n=3, pad=0), dict(in_h=4, in_w=4, kernel_n=1, pad=0),
    dict(in_h=0, in_w=4, kernel_n=3, pad=0), dict(in_h=4, in_w=4, kernel_n=3, pad=-1),
    dict(in_h=4, in_w=4, kernel_n=3, pad=0, c_in=0), dict(in_h=4, in_w=4, kernel_n=3, pad=0, stride=1)])
def test_invalid_specs(kwargs):
    with pytest.raises(P.SpecError):
        P.TransposeConvSpec(**kwargs)


def test_effective_padding_and_subkernel_dims():
    for pad, ep, sw in [(0, 0, False), (1, 0, True), (2, 1, False), (3, 1, True), (4, 2, False), (5, 2, True)]:
        e = P.effective_padding(pad)
        assert (e.pad, e.swap) == (ep, sw)
    with pytest.raises(ValueError):
        P.effective_padding(-1)
    for n in range(2, 10):
        assert P.subkernel_dims(n, 0, 0) == ((n + 1) // 2, (n + 1) // 2)
        assert P.subkernel_dims(n, 0, 1) == ((n + 1) // 2, n // 2)
        assert P.subkernel_dims(n, 1, 0) == (n // 2, (n + 1) // 2)
        assert P.subkernel_dims(n, 1, 1) == (n // 2, n // 2)


def test_mult_counts_match_reference_golden(golden):
    for spec, seg in zip(golden["count_specs"], golden["count_seg"]):
        h, w, n, p, ci, co = (int(v) for v in spec)
        got = P.mult_count_segregated(P.TransposeConvSpec(h, w, n, p, ci, co))
        assert got == int(seg)


def test_mult_count_matches_parity_enumeration():
    # analysis test_parity_enumeration_oracle: tap (u, v) live iff x+u-P, y+v-P even
    for nh, n, pad in [(4, 5, 0), (3, 3, 1), (5, 4, 2), (2, 2, 3), (4, 7, 1)]:
        out_h = 2 * nh + 2 * pad - n
        total = 0
        for x in range(out_h):
            lu = sum(1 for u in range(n) if (x + u - pad) % 2 == 0)
            for y in range(out_h):
                total += lu * sum(1 for v in range(n) if (y + v - pad) % 2 == 0)
        assert P.mult_count_segregated(P.TransposeConvSpec(nh, nh, n, pad)) == total


def test_prepare_validation_precedes_device():
    with pytest.raises(P.ShapeError):
        P.PreparedLayer(np.ones((1, 1, 2, 3), np.float32), 1)
    with pytest.raises(P.ShapeError):
        P.PreparedLayer(np.ones((1, 1, 1, 1), np.float32), 1)
    with pytest.raises(P.ShapeError):
        P.PreparedLayer(np.ones((1, 1, 3, 3), np.int32), 1)
    with pytest.raises(P.SpecError):
        P.PreparedLayer(np.ones((1, 1, 3, 3), np.float32), -1)
    with pytest.raises(ValueError):
        P.PreparedLayer(np.ones((1, 1, 3, 3), np.float32), 0, engine="fastest")


def test_segregate_validation_precedes_device():
    with pytest.raises(P.ShapeError):
        P.segregate_kernel(np.ones((1, 1), np.float32))
    with pytest.raises(P.ShapeError):
        P.segregate_kernel(np.ones((2, 3), np.float32))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        P.layer_forward(np.ones((1, 4, 4), np.float32), np.ones((1, 1, 3, 3), np.float32), 1)


def test_c_abi_error_codes():
    lib = _lib.lib()
    a, b = ctypes.c_int(), ctypes.c_int()
    assert lib.segb_output_dims(1, 1, 3, 0, ctypes.byref(a), ctypes.byref(b)) == _lib.SEGB_ERR_SPEC
    assert "not >= 1" in _lib.last_error()
    assert lib.segb_output_dims(28, 28, 3, 1, ctypes.byref(a), ctypes.byref(b)) == 0
    assert (a.value, b.value) == (55, 55)
    assert lib.segb_mult_count_segregated(1, 1, 3, 0, 1, 1) == -1
    h = ctypes.c_void_p()
    assert lib.segb_prepare(None, 0, 1, 1, 3, 0, 7, 0, None, ctypes.byref(h)) == _lib.SEGB_ERR_VALUE
    assert lib.segb_forward(None, None, 0, 1, 4, 4, None, 0, 0, 0, None) == _lib.SEGB_ERR_VALUE


# analysis.py:60-82 memory_savings_bytes, pinned to the reference's own figures
# (/root/reference/pkg/tests/test_analysis.py:99-125: the paper's Table 4 bytes, pad 2, fp32)
@pytest.mark.parametrize("side,channels,expected", [
    (4, 1024, 495_616), (8, 512, 739_328), (16, 256, 1_254_400), (32, 128, 2_298_368),
    (4, 512, 247_808), (8, 256, 369_664), (4, 2048, 991_232), (8, 1024, 1_478_656),
    (16, 512, 2_508_800), (32, 256, 4_596_736), (64, 128, 8_786_432), (128, 64, 17_172_736)])
def test_memory_savings_gan_layers(side, channels, expected):
    assert P.memory_savings_bytes(side, side, 2, channels) == expected


def test_memory_savings_image_pipeline_and_errors():
    assert P.memory_savings_bytes(224, 224, 2, 3, "upsampled_minus_input") == 1_827_900
    with pytest.raises(P.SpecError):
        P.memory_savings_bytes(0, 4, 2, 3)
    with pytest.raises(P.SpecError):
        P.memory_savings_bytes(4, 4, -1, 3)
    with pytest.raises(ValueError):
        P.memory_savings_bytes(4, 4, 2, 3, "nope")


def test_stack_c_abi_validation():
    lib = _lib.lib()
    v = ctypes.c_int64()
    assert lib.segb_stack_workspace_bytes(None, 0, 1, 4, 4, _lib.BF16, ctypes.byref(v)) == _lib.SEGB_ERR_VALUE
    assert "at least one layer" in _lib.last_error()
    arr = (ctypes.c_void_p * 2)(None, None)
    assert lib.segb_stack_workspace_bytes(arr, 2, 1, 4, 4, _lib.BF16, ctypes.byref(v)) == _lib.SEGB_ERR_VALUE
    assert lib.segb_stack_forward(arr, 2, None, 0, 1, 4, 4, None, 0, 0, None, 0, None) == _lib.SEGB_ERR_VALUE
    assert lib.segb_stack_forward(arr, 2, None, 0, 0, 4, 4, None, 0, 0, None, 0, None) == _lib.SEGB_ERR_SHAPE
