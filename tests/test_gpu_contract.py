"""GPU tests of the boundary's contract (include/segb200.h):

  * the instrumented scalar engines (engines.py:353-406) on the device equal the reference's
    outputs and counters bit for bit (tests/golden cnt*, made from the reference itself);
  * forward never allocates: the scratch is sized by segb_forward_workspace_bytes and passed in
    (K2 / K3b need none), segb_forward without a reserved workspace refuses a K3 shape;
  * a freshly prepared layer is capturable into a CUDA graph from its very first forward, on
    every kernel family, and the replay equals the eager call bitwise;
  * a layout that prepare did not build is refused inside a capture instead of being recorded;
  * a host `out=` tensor is complete when forward returns.
"""

import ctypes

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


def test_counted_engines_known_counts():
    """test_engines.py:198-233 of the reference: 225 / 64 multiplications, 9 writes"""
    f32 = np.float32
    out, c = P.transpose_conv_reference_counted(np.ones((4, 4), f32), np.ones((5, 5), f32), 0)
    assert out.shape == (3, 3) and out.dtype == np.float64
    assert (c.mults, c.writes) == (225, 9)
    subs = P.segregate_kernel(np.ones((5, 5), f32))
    out, c = P.transpose_conv_segregated_counted(np.ones((4, 4), f32), subs, 0)
    assert out.shape == (3, 3)
    assert (c.mults, c.writes) == (4 * 9 + 2 * 6 + 2 * 6 + 1 * 4, 9)
    assert isinstance(c, P.EngineCounters)


def test_counted_engines_bitwise_golden(golden):
    for i in range(int(golden["n_cnt"])):
        m, k, pad = golden[f"cnt{i}_map"], golden[f"cnt{i}_kernel"], int(golden[f"cnt{i}_pad"])
        rm, rw, sm, sw = (int(v) for v in golden[f"cnt{i}_counts"])
        ref, cr = P.transpose_conv_reference_counted(m, k, pad)
        seg, cs = P.transpose_conv_segregated_counted(m, P.segregate_kernel(k), pad)
        assert np.array_equal(ref, golden[f"cnt{i}_ref"]), i
        assert np.array_equal(seg, golden[f"cnt{i}_seg"]), i
        assert (cr.mults, cr.writes, cs.mults, cs.writes) == (rm, rw, sm, sw), i


def test_counted_engines_errors():
    with pytest.raises(P.SpecError):
        P.transpose_conv_reference_counted(np.ones((1, 1), np.float32), np.ones((5, 5), np.float32), 0)
    with pytest.raises(P.ShapeError):
        P.transpose_conv_reference_counted(np.ones((3,), np.float32), np.ones((3, 3), np.float32), 0)


# (c_in, c_out, n, pad, batch, h, w, compute, x dtype) per kernel family
FAMILIES = {
    "K2 fp32": (3, 1, 5, 2, 2, 21, 17, "fp32", "float32"),
    "K2 fp64": (2, 2, 3, 1, 2, 9, 11, "fp64", "float64"),
    "K3 bf16": (256, 128, 4, 2, 2, 16, 16, "bf16", "bfloat16"),
    "K3p bf16": (256, 128, 4, 2, 2, 32, 32, "bf16", "bfloat16"),
    "K3b bf16": (64, 64, 4, 2, 2, 64, 64, "bf16", "bfloat16"),
    "K3c bf16": (128, 3, 4, 2, 2, 32, 32, "bf16", "bfloat16"),
    "K3 3xTF32": (64, 32, 4, 2, 2, 16, 16, "fp32", "float32"),
}


def _layer_and_input(fam, seed=5):
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    ci, co, n, pad, b, h, w, compute, xdt = FAMILIES[fam]
    bank = O.gen_kernel_bank(ci, co, n, seed)
    layer = P.prepare_layer(bank if compute != "fp64" else bank.astype(np.float64), pad, compute=compute)
    x = device_unit_floats((b, ci, h, w), seed + 1, dtype=torch.float32 if xdt == "float64" else getattr(torch, xdt))
    return layer, x.to(getattr(torch, xdt))


@pytest.mark.parametrize("fam", sorted(FAMILIES))
def test_fresh_layer_captures_into_a_graph(fam):
    """no warm-up call: the first forward of a just-prepared layer is recorded into a CUDA
    graph (prepare built every layout; the workspace comes from the graph's pool)"""
    import torch
    layer, x = _layer_and_input(fam)
    oh, ow = layer.output_shape(x.shape[2], x.shape[3])
    y_graph = torch.full((x.shape[0], layer.c_out, oh, ow), float("nan"), dtype=x.dtype, device=x.device)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer.forward(x, out=y_graph)
    g.replay()
    torch.cuda.synchronize()
    y_eager = layer.forward(x)
    torch.cuda.synchronize()
    assert not torch.isnan(y_graph).any()
    assert torch.equal(y_graph, y_eager)


def test_workspace_contract():
    import torch
    from paper_2502_20493_b200 import _lib
    k3b, xb = _layer_and_input("K3b bf16")
    assert k3b.select_path(_lib.BF16, 2, 64, 64) == "igemm"
    assert k3b.workspace_bytes(2, 64, 64) == 0
    k3, x = _layer_and_input("K3 bf16")
    need = k3.workspace_bytes(2, 16, 16)
    assert need >= 2 * 256 * 16 * 16 * 2  # the channels-last bf16 copy of x
    k2, x2 = _layer_and_input("K2 fp32")
    assert k2.workspace_bytes(2, 21, 17) == 0
    # segb_forward (layer-owned workspace) refuses until the workspace is reserved
    lib = _lib.lib()
    y = torch.empty((2, 128, 32, 32), dtype=torch.bfloat16, device="cuda")
    args = (k3._handle, x.data_ptr(), _lib.BF16, 2, 16, 16, y.data_ptr(), _lib.BF16, -1, 0,
            torch.cuda.current_stream().cuda_stream)
    assert lib.segb_forward(*args) == _lib.SEGB_ERR_VALUE
    assert str(need) in _lib.last_error()
    _lib.check(lib.segb_layer_reserve_workspace(k3._handle, need))
    _lib.check(lib.segb_forward(*args))
    torch.cuda.synchronize()
    assert torch.equal(y, k3.forward(x))
    # segb_forward_ws with a short workspace is refused
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    rc = lib.segb_forward_ws(k3._handle, x.data_ptr(), _lib.BF16, 2, 16, 16, y.data_ptr(), _lib.BF16, -1, 0,
                             ws.data_ptr(), need - 1, torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.SEGB_ERR_VALUE
    v = ctypes.c_int64()
    _lib.check(lib.segb_forward_workspace_bytes(k3._handle, _lib.BF16, 2, 16, 16, _lib.BF16, -1, 0,
                                                ctypes.byref(v)))
    assert v.value == need


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")  # the refused capture records nothing
def test_unbuilt_layout_refused_inside_capture():
    """an fp32-prepared layer fed fp64 needs the fp64 direct layout, which prepare did not
    build: inside a capture that is an error, outside it is built once (synchronously)"""
    import torch
    bank = O.gen_kernel_bank(3, 1, 5, 5)
    layer = P.prepare_layer(bank, 2)
    x64 = torch.rand((1, 3, 21, 17), dtype=torch.float64, device="cuda")
    y = torch.empty((1, 1, 41, 33), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(ValueError, match="capture"):
        with torch.cuda.graph(g):
            layer.forward(x64, out=y)
    torch.cuda.synchronize()
    out = layer.forward(x64).cpu().numpy()
    ref = O.forward_segregated(x64.cpu().numpy()[0], bank.astype(np.float64), 2)
    assert O.compare(out[0], ref, 0, 1e-12)["passed"]


def test_host_out_is_complete_on_return():
    import torch
    layer, x = _layer_and_input("K3b bf16")
    oh, ow = layer.output_shape(64, 64)
    for _ in range(3):
        host = torch.full((2, 64, oh, ow), float("nan"), dtype=torch.bfloat16).pin_memory()
        layer.forward(x, out=host)
        assert not torch.isnan(host).any()  # read right away, no synchronize
    assert torch.equal(host, layer.forward(x).cpu())


def test_in_flight_host_copies_then_wait():
    """non_blocking host outputs of consecutive pipelined forwards: the copies overlap the next
    call; after wait_host_copies() and a synchronize every output is complete and equal to the
    blocking result"""
    import torch
    layer, x = _layer_and_input("K3b bf16")
    xh = torch.cat([x] * 4).cpu().pin_memory()  # a batch the host pipeline takes
    oh, ow = layer.output_shape(64, 64)
    outs = [torch.full((xh.shape[0], 64, oh, ow), float("nan"), dtype=torch.bfloat16).pin_memory() for _ in range(3)]
    for o in outs:
        layer.forward(xh, out=o, non_blocking=True)
    P.wait_host_copies(x.device)
    done = torch.cuda.Event()
    done.record()
    done.synchronize()
    ref = layer.forward(xh)
    for o in outs:
        assert torch.equal(o, ref)


@pytest.mark.parametrize("ci,co,h,batch,compute", [(2048, 1024, 4, 64, "fp32"), (1024, 512, 4, 96, "bf16"),
                                                    (64, 64, 128, 6, "fp32")])
def test_host_pipeline_bitwise_whole_batch(ci, co, h, batch, compute):
    """the pipelined host path picks chunks that dispatch as the whole batch: bitwise the
    device-resident whole-batch forward (ebgan_l2-like layers change tile configuration at
    small batches)"""
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    tdt = torch.bfloat16 if compute == "bf16" else torch.float32
    layer = P.prepare_layer(device_unit_floats((ci, co, 4, 4), 3), 2, compute=compute)
    xd = device_unit_floats((batch, ci, h, h), 4, dtype=tdt)
    want = layer.forward(xd).cpu()
    xh = xd.cpu().pin_memory()
    oh, ow = layer.output_shape(h, h)
    out = torch.empty((batch, co, oh, ow), dtype=want.dtype).pin_memory()
    layer.forward(xh, out=out)
    assert torch.equal(out, want)
