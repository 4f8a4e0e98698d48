"""GPU tests of device-resident layer stacks (paper_2502_20493_b200/stack.py).

A stack must equal the layer-by-layer chain of PreparedLayer.forward calls whose
intermediates are rounded to the stack's intermediate dtype -- bitwise, since each layer
runs the same kernel with the same accumulation order -- and, through that chain, the
reference oracle applied layer after layer (fp32: the reference's rel 1e-5 / abs 1e-6 gate
per layer, compounded over the chain).
"""

import numpy as np
import pytest

import paper_2502_20493_b200 as P
from oracle import segconv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _chain(layers, x, inter_dtype):
    """layer-by-layer PreparedLayer.forward on the device, intermediates in inter_dtype"""
    for i, L in enumerate(layers):
        last = i + 1 == len(layers)
        x = L.forward(x, out_dtype=None if last else inter_dtype)
    return x


# GAN-generator-like bf16 stack: K3 (tcgen05) and K3b layers, the DCGAN tail on K3c (c_out 3)
BF16_STACK = [(256, 128, 4, 2), (128, 64, 4, 2), (64, 64, 4, 2), (64, 3, 4, 2)]  # (c_in, c_out, n, pad)


def test_bf16_stack_equals_layer_chain():
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    layers = [P.prepare_layer(O.gen_kernel_bank(ci, co, n, 11 + i), pad, compute="bf16")
              for i, (ci, co, n, pad) in enumerate(BF16_STACK)]
    stack = P.prepare_stack(layers)
    assert stack.inter_dtype == "bf16"
    x = device_unit_floats((4, 256, 8, 8), 5, dtype=torch.bfloat16)
    y = stack.forward(x)
    ref = _chain(layers, x, torch.bfloat16)
    assert y.shape == (4, 3, 128, 128) and y.dtype == ref.dtype
    assert torch.equal(y, ref)


def test_bf16_stack_host_batch_graph_replay():
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    layers = [P.prepare_layer(O.gen_kernel_bank(ci, co, n, 21 + i), pad, compute="bf16")
              for i, (ci, co, n, pad) in enumerate(BF16_STACK[:3])]
    stack = P.prepare_stack(layers)
    xd = device_unit_floats((2, 256, 8, 8), 9, dtype=torch.bfloat16)
    want = stack.forward(xd).cpu()
    xh = xd.cpu().pin_memory()
    oh = torch.empty(tuple(want.shape), dtype=want.dtype).pin_memory()
    for _ in range(2):  # capture, then replay
        oh.zero_()
        stack.forward(xh, out=oh)
        assert torch.equal(oh, want)
    assert len(stack._graphs) == 1
    assert torch.equal(stack.forward(xh), want)  # host in -> host tensor out


def test_stack_host_batch_chunk_pipeline():
    """a host batch whose output is large enough for the chunked pipeline (copy-out of chunk k-1
    beside the chain of chunk k; chunks that dispatch as the whole batch): bitwise the whole-batch
    device chain"""
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    layers = [P.prepare_layer(O.gen_kernel_bank(ci, co, n, 41 + i), pad, compute="bf16")
              for i, (ci, co, n, pad) in enumerate(BF16_STACK[:3])]
    stack = P.prepare_stack(layers)
    xd = device_unit_floats((64, 256, 8, 8), 13, dtype=torch.bfloat16)
    import paper_2502_20493_b200.stack as S
    S._STACK_PIPELINE_MIN_BYTES = 8 << 20  # (the 33 MB output of this test is below the default)
    want = stack.forward(xd).cpu()
    xh = xd.cpu().pin_memory()
    oh = torch.empty(tuple(want.shape), dtype=want.dtype).pin_memory()
    for _ in range(2):
        oh.fill_(float("nan"))
        stack.forward(xh, out=oh)
        assert torch.equal(oh, want)
    assert stack._pipeline_chunk(64, 8, 8, torch.bfloat16, torch.bfloat16) > 0
    assert any(k[0] == "chunk" for k in stack._graphs)


def test_fp32_stack_matches_oracle_chain():
    """low-channel fp32 chain on the direct kernel, odd kernels and an odd P (the swap)"""
    import torch
    specs = [(2, 3, 3, 1), (3, 2, 5, 2), (2, 1, 4, 3)]
    banks = [O.gen_kernel_bank(ci, co, n, 31 + i) for i, (ci, co, n, pad) in enumerate(specs)]
    layers = [P.prepare_layer(bk, pad) for bk, (ci, co, n, pad) in zip(banks, specs)]
    stack = P.prepare_stack(layers)
    assert stack.inter_dtype == "fp32"
    x = O.unit_floats(3 * 2 * 9 * 7, 41).reshape(3, 2, 9, 7)
    y = stack.forward(torch.from_numpy(x).cuda())
    assert torch.equal(y, _chain(layers, torch.from_numpy(x).cuda(), None))
    ref = []
    for xi in x.astype(np.float64):
        for bk, (ci, co, n, pad) in zip(banks, specs):
            xi = O.forward_segregated(xi, bk.astype(np.float64), pad)
        ref.append(xi)
    ref = np.stack(ref)
    assert y.shape == ref.shape
    rep = O.compare(y.cpu().numpy(), ref, 3e-5, 3e-6)  # three chained fp32 layers
    assert rep["passed"], rep


def test_stack_validation():
    layers = [P.prepare_layer(O.gen_kernel_bank(2, 3, 3, 1), 1), P.prepare_layer(O.gen_kernel_bank(4, 1, 3, 2), 1)]
    with pytest.raises(P.ShapeError):
        P.prepare_stack(layers)
    with pytest.raises(ValueError):
        P.prepare_stack([])
    import torch
    ok = P.prepare_stack(layers[:1])
    with pytest.raises(P.ShapeError):
        ok.forward(torch.zeros((1, 5, 4, 4), device="cuda"))
