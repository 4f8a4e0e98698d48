"""K2p, the paired FFMA2 direct kernel for low-channel fp32 layers (csrc/direct_pair.cuh; fp32 x with
W % 4 == 0 takes its TMA-staged variant): bitwise equal to K2 (same per-element rule and summation order; SEGB200_DIRECT_PAIR=0 selects K2) over
kernel sides (4, 5), paddings (both swap parities), channel counts, odd batches (the last sample
unpaired), odd and tiny spatial sizes, and within the reference's fp32 gate of the oracle
(rel 1e-5 / abs 1e-6, /root/reference/pkg/tests/test_acceptance.py:31)."""

import os

import numpy as np
import pytest

import paper_2502_20493_b200 as P
from oracle import segconv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


def _forward_both(torch, layer, x):
    y_pair = layer.forward(x)
    os.environ["SEGB200_DIRECT_PAIR"] = "0"
    try:
        path_k2 = layer.describe_path(x.shape[0], x.shape[2], x.shape[3])
        y_k2 = layer.forward(x)
    finally:
        del os.environ["SEGB200_DIRECT_PAIR"]
    assert path_k2.startswith("K2 ")
    return y_pair, y_k2


CASES = [  # (batch, c_in, c_out, n, pad, h, w)
    (1, 3, 1, 5, 2, 37, 53), (3, 3, 1, 5, 2, 64, 64), (2, 3, 3, 4, 1, 31, 17), (5, 1, 1, 4, 0, 28, 28),
    (4, 1, 1, 5, 1, 28, 28), (4, 1, 1, 4, 2, 28, 28), (2, 3, 2, 4, 0, 9, 11), (3, 5, 3, 4, 3, 20, 33),
    (2, 7, 1, 5, 4, 16, 16), (7, 3, 1, 4, 2, 1, 1), (2, 3, 3, 5, 2, 66, 130), (6, 2, 2, 5, 3, 5, 40),
    # W % 4 == 0: the TMA-staged variant, boxes past every edge of small images; n = 3 runs only there
    (2, 3, 1, 5, 3, 5, 4), (3, 2, 2, 4, 1, 3, 8), (1, 3, 3, 5, 0, 9, 12), (5, 1, 1, 4, 2, 20, 132),
    (3, 1, 1, 3, 0, 28, 28), (4, 1, 1, 3, 1, 28, 28), (2, 3, 2, 3, 2, 30, 36), (3, 3, 3, 3, 3, 7, 8),
]


@pytest.mark.parametrize("batch,c_in,c_out,n,pad,h,w", CASES)
def test_pair_bitwise_k2_and_oracle(torch, batch, c_in, c_out, n, pad, h, w):
    bank = O.gen_kernel_bank(c_in, c_out, n, 11 + n)
    layer = P.prepare_layer(bank, pad)
    x = torch.from_numpy(O.unit_floats(batch * c_in * h * w, 5 + h).reshape(batch, c_in, h, w)).cuda()
    assert layer.describe_path(batch, h, w).startswith("K2p ")
    y_pair, y_k2 = _forward_both(torch, layer, x)
    assert torch.equal(y_pair, y_k2)
    ref = O.forward_segregated_batch(x.cpu().numpy().astype(np.float64), bank.astype(np.float64), pad)
    assert O.compare(y_pair.cpu().numpy(), ref, 1e-5, 1e-6)["passed"]


def test_pair_dataset_shape_bitwise(torch):
    """ds512_k5 at a small batch: interior fast loads and the border path in one launch"""
    bank = O.gen_kernel_bank(3, 1, 5, 3)
    layer = P.prepare_layer(bank, 2)
    x = torch.rand((3, 3, 512, 512), device="cuda")
    y_pair, y_k2 = _forward_both(torch, layer, x)
    assert torch.equal(y_pair, y_k2)


def test_pair_not_taken_outside_its_range(torch):
    """wide layers, n outside 3..5, bf16 compute and the reference engine stay on their kernels"""
    for c_in, c_out, n, compute in [(3, 4, 4, "fp32"), (3, 1, 7, "fp32"), (3, 1, 5, "bf16")]:
        layer = P.prepare_layer(O.gen_kernel_bank(c_in, c_out, n, 1), 2, compute=compute)
        assert not layer.describe_path(2, 16, 16).startswith("K2p")
    # n = 3 only on the TMA-staged variant (W % 4 == 0)
    layer = P.prepare_layer(O.gen_kernel_bank(3, 1, 3, 1), 2)
    assert layer.describe_path(2, 16, 18).startswith("K2 ") and layer.describe_path(2, 16, 16).startswith("K2p")
    layer = P.prepare_layer(O.gen_kernel_bank(3, 1, 5, 1), 2, engine="reference")
    assert not layer.describe_path(2, 16, 16).startswith("K2p")


@pytest.mark.parametrize("batch,c_in,c_out,n,pad,h,w", [(3, 3, 1, 5, 2, 37, 53), (5, 2, 3, 4, 1, 9, 70),
                                                         (1, 3, 2, 4, 3, 1, 1)])
def test_pair_writes_exactly_the_output(torch, batch, c_in, c_out, n, pad, h, w):
    """every output element written once, nothing around it: y is a window of a NaN-filled buffer"""
    layer = P.prepare_layer(O.gen_kernel_bank(c_in, c_out, n, 2), pad)
    oh, ow = layer.output_shape(h, w)
    count, guard = batch * c_out * oh * ow, 4096
    buf = torch.full((count + 2 * guard,), float("nan"), device="cuda")
    y = buf[guard:guard + count].view(batch, c_out, oh, ow)
    x = torch.rand((batch, c_in, h, w), device="cuda")
    layer.forward(x, out=y)
    torch.cuda.synchronize()
    assert not torch.isnan(y).any()
    assert torch.isnan(buf[:guard]).all() and torch.isnan(buf[guard + count:]).all()


@pytest.mark.parametrize("batch,c_in,c_out,n,pad,h,w", [(2, 128, 3, 4, 2, 32, 32), (3, 96, 2, 5, 1, 12, 20),
                                                         (4, 200, 1, 3, 3, 9, 16)])
def test_pair_weights_in_shared_memory(torch, batch, c_in, c_out, n, pad, h, w):
    """more weights than the kernel parameter holds (dcgan_l5: 128 x 3 x 16): the TMA-staged K2p
    reads them from shared memory; bitwise K2 and within the oracle's gate"""
    bank = O.gen_kernel_bank(c_in, c_out, n, 21 + n)
    layer = P.prepare_layer(bank, pad)
    x = torch.from_numpy(O.unit_floats(batch * c_in * h * w, 3 + h).reshape(batch, c_in, h, w)).cuda()
    assert "weights in shared memory" in layer.describe_path(batch, h, w, path="direct")
    y_pair = layer.forward(x, path="direct")
    os.environ["SEGB200_DIRECT_PAIR"] = "0"
    try:
        y_k2 = layer.forward(x, path="direct")
    finally:
        del os.environ["SEGB200_DIRECT_PAIR"]
    assert torch.equal(y_pair, y_k2)
    ref = O.forward_segregated_batch(x.cpu().numpy().astype(np.float64), bank.astype(np.float64), pad)
    assert O.compare(y_pair.cpu().numpy(), ref, 1e-5, 1e-6)["passed"]

