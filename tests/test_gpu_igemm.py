"""GPU parity of K3 (tcgen05 implicit GEMM, bf16 operands, fp32 accumulation).

Gates (stated tolerances for the bf16 tensor-core path):
  * fp32 output vs the fp64 oracle evaluated on the *same bf16-rounded* inputs
    and weights: rel 1e-4 / abs 1e-5 (only accumulation order differs; products
    of bf16 values are exact in fp32);
  * bf16 output vs the same oracle: rel 2^-7 (one bf16 rounding of the result
    plus accumulation), abs 1e-3 * max|ref|;
  * vs the fp32 reference on the unrounded fp32 inputs: rel 1.6e-2,
    abs 1e-2 * max|ref| (SURVEY 7.4 recommendation);
  * igemm and the direct bf16 kernel agree to rel 1e-4 (same arithmetic contract).
"""

import numpy as np
import pytest

import paper_2502_20493_b200 as P
from oracle import segconv_oracle as O

pytestmark = pytest.mark.gpu

CASES = [  # name, h, w, c_in, n, c_out, pad, batch
    ("ebgan_l7", 128, 128, 64, 4, 64, 2, 2),
    ("ebgan_l6", 64, 64, 128, 4, 64, 2, 2),
    ("ebgan_l5", 32, 32, 256, 4, 128, 2, 2),
    ("ebgan_l4", 16, 16, 512, 4, 256, 2, 2),
    ("ebgan_l3", 8, 8, 1024, 4, 512, 2, 4),
    ("ebgan_l2", 4, 4, 2048, 4, 1024, 2, 8),
    ("dcgan_l2_b3", 4, 4, 1024, 4, 512, 2, 3),   # partial last tile
    ("odd_pad", 16, 16, 64, 2, 32, 1, 2),        # swap rule on the tensor-core path
    ("n6_p3", 8, 8, 64, 6, 96, 3, 4),
    ("n2_p1", 32, 64, 96, 2, 160, 1, 2),
    ("dcgan_l5_cout3", 32, 32, 128, 4, 3, 2, 2),  # K3c scatter GEMM (N = 16 taps x 3)
    ("cout48", 16, 16, 64, 4, 48, 2, 2),
    # K3c (input-stationary scatter GEMM + gather): odd kernels, odd P, tiles that straddle
    # images and a partial last tile, 1..4 channel blocks, N up to 256
    ("scatter_n3_p1", 16, 16, 64, 3, 2, 1, 3),
    ("scatter_n5_p2_tail", 8, 8, 192, 5, 4, 2, 3),
    ("scatter_n4_p0_n256", 16, 8, 256, 4, 16, 0, 2),
    ("scatter_n2_p3", 8, 16, 64, 2, 1, 3, 5),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _inputs(h, w, ci, n, co, b, seed):
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    x = device_unit_floats((b, ci, h, w), seed, dtype=torch.bfloat16)
    bank = O.gen_kernel_bank(ci, co, n, seed + 1)
    return x, bank


@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b", CASES)
def test_igemm_matches_oracle(name, h, w, ci, n, co, pad, b):
    import torch
    x, bank = _inputs(h, w, ci, n, co, b, 1000 + h + ci)
    layer = P.prepare_layer(bank, pad, compute="bf16")
    assert layer.select_path(2, b, h, w) == "igemm", name
    y32 = layer.forward(x, path="igemm", out_dtype=torch.float32).cpu().numpy()
    xr = x.float().cpu().numpy().astype(np.float64)
    br = O.bf16_round(bank).astype(np.float64)
    ref = O.forward_segregated_batch(xr, br, pad)
    rep = O.compare(y32, ref, 1e-4, 1e-5)
    assert rep["passed"], (name, rep)
    yb = layer.forward(x, path="igemm").float().cpu().numpy()
    repb = O.compare(yb, ref, 2 ** -7, 1e-3 * float(np.abs(ref).max()))
    assert repb["passed"], (name, repb)
    # same arithmetic contract as the direct bf16 kernel
    yd = layer.forward(x, path="direct", out_dtype=torch.float32).cpu().numpy()
    assert O.compare(y32, yd.astype(np.float64), 1e-4, 1e-5)["passed"], name


def test_igemm_vs_fp32_reference_loose():
    import torch
    h, w, ci, n, co, pad, b = 32, 32, 128, 4, 64, 2, 2
    rng = np.random.default_rng(5)
    x32 = rng.random((b, ci, h, w)).astype(np.float32)
    bank = rng.random((ci, co, n, n)).astype(np.float32)
    layer = P.prepare_layer(bank, pad, compute="bf16")
    y = layer.forward(torch.from_numpy(x32).cuda(), path="igemm").cpu().numpy()  # fp32 in -> bf16 staged
    ref = O.forward_segregated_batch(x32.astype(np.float64), bank.astype(np.float64), pad)
    rep = O.compare(y, ref, 1.6e-2, 1e-2 * float(np.abs(ref).max()))
    assert rep["passed"], rep


def test_igemm_deterministic_and_batch_invariant():
    import torch
    h, w, ci, n, co, pad = 16, 16, 128, 4, 64, 2
    x, bank = _inputs(h, w, ci, n, co, 6, 77)
    layer = P.prepare_layer(bank, pad, compute="bf16")
    a = layer.forward(x, path="igemm")
    b = layer.forward(x, path="igemm")
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    # a shard of the batch computes bitwise the same samples (multi-GPU sharding contract)
    c = layer.forward(x[2:4].contiguous(), path="igemm")
    assert torch.equal(a[2:4].view(torch.int16), c.view(torch.int16))


def test_igemm_write_once_guard():
    import torch
    h, w, ci, n, co, pad, b = 8, 8, 64, 4, 32, 2, 3
    x, bank = _inputs(h, w, ci, n, co, b, 91)
    layer = P.prepare_layer(bank, pad, compute="bf16")
    oh, ow = layer.output_shape(h, w)
    total = b * co * oh * ow
    buf = torch.full((4096 + total + 4096,), float("nan"), device="cuda")
    y = buf[4096:4096 + total].view(b, co, oh, ow)
    layer.forward(x, out=y, path="igemm")
    torch.cuda.synchronize()
    assert not torch.isnan(y).any()
    assert torch.isnan(buf[:4096]).all() and torch.isnan(buf[4096 + total:]).all()


ROWS_CASES = [  # K3b row-streaming variant: class grid cols % 128 == 0, c_out <= 64
    ("ebgan_l7", 128, 128, 64, 4, 64, 2, 3),
    ("rows_msub2", 32, 256, 64, 4, 32, 2, 2),
    ("rows_kb2_n16", 16, 128, 128, 4, 16, 2, 2),
    ("rows_odd_pad_n2", 16, 128, 64, 2, 32, 1, 2),
    ("rows_n6_p3", 8, 128, 64, 6, 16, 3, 2),
    ("rows_cin_tail", 16, 128, 40, 4, 48, 2, 2),
    ("rows_m64_l6", 64, 64, 128, 4, 64, 2, 2),      # M=64 rows, 2-way output-channel split
    ("rows_m64_kb1", 32, 64, 64, 4, 32, 2, 2),      # M=64 rows, weights resident unsplit
    ("rows_m64_msub2", 8, 128 + 64 - 64, 128, 4, 64, 2, 2),
    ("rows_m64_pair_b4", 32, 64, 128, 4, 32, 2, 4),  # 2-SM CTA pairs over the batch halves
    ("rows_m64_odd_batch", 32, 64, 128, 4, 64, 2, 3),  # odd batch: no pairing
]


@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b", ROWS_CASES)
def test_igemm_rows_variant(name, h, w, ci, n, co, pad, b, monkeypatch):
    """K3b writes bf16 (TMA-stored); gate: one bf16 rounding of an fp32-accumulated result."""
    import torch
    x, bank = _inputs(h, w, ci, n, co, b, 500 + w + ci)
    xr = x.float().cpu().numpy().astype(np.float64)
    br = O.bf16_round(bank).astype(np.float64)
    ref = O.forward_segregated_batch(xr, br, pad)
    layer = P.prepare_layer(bank, pad, compute="bf16")
    assert layer.select_path(2, b, h, w) == "igemm", name
    yb = layer.forward(x, path="igemm").float().cpu().numpy()
    rep = O.compare(yb, ref, 2 ** -8 + 1e-4, 1e-6 * float(np.abs(ref).max()))
    assert rep["passed"], (name, rep)
    # the fp32-output request goes through K3 where eligible, else the direct kernel
    path = "igemm"
    monkeypatch.setenv("SEGB200_IGEMM_GENERIC", "1")
    try:
        y32 = layer.forward(x, path=path, out_dtype=torch.float32).cpu().numpy()
    except NotImplementedError:
        y32 = layer.forward(x, path="direct", out_dtype=torch.float32).cpu().numpy()
    assert O.compare(y32, ref, 1e-4, 1e-5)["passed"], name
    assert O.compare(yb, y32.astype(np.float64), 2 ** -8 + 1e-4, 1e-6 * float(np.abs(ref).max()))["passed"], name


TF32_CASES = [  # fp32 layers on tensor cores (3xFP16 where c_in >= 64, else 3xTF32): the reference's fp32 gate
    ("ebgan_l2", 4, 4, 2048, 4, 1024, 2, 8),
    ("ebgan_l5", 32, 32, 256, 4, 128, 2, 2),
    ("ebgan_l7", 128, 128, 64, 4, 64, 2, 1),
    ("odd_pad_n2", 16, 16, 64, 2, 32, 1, 2),
    ("n6_p3_tail", 8, 8, 40, 6, 96, 3, 4),
]


@pytest.mark.parametrize("mode", ["3xFP16", "3xTF32"])
@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b", TF32_CASES)
def test_igemm_3xtf32_fp32_tolerance(monkeypatch, mode, name, h, w, ci, n, co, pad, b):
    """fp32 compute on the tensor-core path must still meet rel 1e-5 / abs 1e-6 against the
    reference's fp32 engine inputs (oracle evaluated in fp64), in both operand modes
    (SEGB200_FP32_TC=tf32x3 forces 3xTF32 at prepare)."""
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    if mode == "3xTF32":
        monkeypatch.setenv("SEGB200_FP32_TC", "tf32x3")
    x = device_unit_floats((b, ci, h, w), 900 + ci, dtype=torch.float32)
    bank = O.gen_kernel_bank(ci, co, n, 901 + ci)
    layer = P.prepare_layer(bank, pad)  # compute = fp32 (the reference's working precision)
    assert layer.select_path(0, b, h, w) == "igemm", name
    want = mode if (mode == "3xTF32" or ci >= 64) else "3xTF32"
    assert want in layer.describe_path(b, h, w), (name, layer.describe_path(b, h, w))
    y = layer.forward(x, path="igemm").cpu().numpy()
    ref = O.forward_segregated_batch(x.cpu().numpy().astype(np.float64), bank.astype(np.float64), pad)
    rep = O.compare(y, ref, 1e-5, 1e-6)
    assert rep["passed"], (name, rep)
    yd = layer.forward(x, path="direct").cpu().numpy()
    assert O.compare(yd, ref, 1e-5, 1e-6)["passed"], name


def test_scatter_matches_output_stationary_path(monkeypatch):
    """K3c and the output-stationary K3 GEMM compute the same layer (SEGB200_IGEMM_NOSCATTER)."""
    import torch
    h, w, ci, n, co, pad, b = 32, 32, 128, 4, 3, 2, 3
    x, bank = _inputs(h, w, ci, n, co, b, 77)
    layer = P.prepare_layer(bank, pad, compute="bf16")
    ys = layer.forward(x, path="igemm", out_dtype=torch.float32).cpu().numpy()
    monkeypatch.setenv("SEGB200_IGEMM_NOSCATTER", "1")
    yk = layer.forward(x, path="igemm", out_dtype=torch.float32).cpu().numpy()
    assert O.compare(ys, yk.astype(np.float64), 1e-4, 1e-5)["passed"]


@pytest.mark.parametrize("pm", ["0", "1", "2"])
@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b,compute", [
    ("odd_m_tiles", 8, 8, 128, 4, 256, 2, 5, "bf16"),     # 5 x 64 positions: 3 blocks, last pair half empty
    ("pairs_n128", 8, 8, 128, 4, 128, 2, 5, "bf16"),      # 5 x 64 positions: 3 blocks, odd
    ("pairs_n256_p1", 8, 8, 64, 2, 256, 1, 4, "bf16"),    # odd P on the paired path
    ("pairs_tf32", 8, 8, 64, 4, 64, 2, 5, "fp32"),        # 3xTF32 through the pair modes
])
def test_k3_cta_pair_modes(monkeypatch, pm, name, h, w, ci, n, co, pad, b, compute):
    """K3 single-CTA (0), B-multicast pair (1) and 2-SM cta_group::2 pair (2) all match the oracle."""
    import torch
    monkeypatch.setenv("SEGB200_K3_PAIR", pm)
    monkeypatch.setenv("SEGB200_IGEMM_GENERIC", "1")
    monkeypatch.setenv("SEGB200_K3_CP", "0")  # the per-class K3 kernel, not the class-pair one
    x, bank = _inputs(h, w, ci, n, co, b, 4242 + int(pm))
    if compute == "fp32":
        x = x.float()
    layer = P.prepare_layer(bank, pad, compute=compute)
    y = layer.forward(x, path="igemm", out_dtype=torch.float32).cpu().numpy()
    xr = x.float().cpu().numpy().astype(np.float64)
    br = (O.bf16_round(bank) if compute == "bf16" else bank).astype(np.float64)
    ref = O.forward_segregated_batch(xr, br, pad)
    tol = (1e-4, 1e-5) if compute == "bf16" else (1e-5, 1e-6)
    rep = O.compare(y, ref, *tol)
    assert rep["passed"], (name, pm, rep)


@pytest.mark.parametrize("pair", ["0", "1", "4"])
@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b", [
    ("l6_like", 64, 64, 128, 4, 64, 2, 4),
    ("kb1_c32", 32, 64, 64, 4, 32, 2, 6),
    ("l7_like", 32, 128, 64, 4, 64, 2, 4),         # "4": M=256 pairs (natural weight halves)
    ("kb2_c32_128", 32, 128, 128, 4, 32, 2, 4),
])
def test_rows_cta_pair_on_off(monkeypatch, pair, name, h, w, ci, n, co, pad, b):
    """K3b as 2-SM CTA pairs (cta_group::2: M=128 for 64-wide rows, M=256 for 128-wide ones with
    SEGB200_ROWS_PAIR=4) or single CTAs."""
    import torch
    monkeypatch.setenv("SEGB200_ROWS_PAIR", pair)
    x, bank = _inputs(h, w, ci, n, co, b, 900 + int(pair))
    layer = P.prepare_layer(bank, pad, compute="bf16")
    yb = layer.forward(x, path="igemm").float().cpu().numpy()
    ref = O.forward_segregated_batch(x.float().cpu().numpy().astype(np.float64),
                                     O.bf16_round(bank).astype(np.float64), pad)
    rep = O.compare(yb, ref, 2 ** -8 + 1e-4, 1e-6 * float(np.abs(ref).max()))
    assert rep["passed"], (name, pair, rep)


@pytest.mark.parametrize("cp", ["0", "1"])
@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b", [
    ("n4_p2", 16, 16, 128, 4, 128, 2, 3),       # shared middle window, odd batch (half-empty last pair)
    ("n4_p1_swap", 9, 17, 64, 4, 48, 1, 2),      # odd P: both column classes read every window
    ("n2_p2_noshare", 7, 15, 64, 2, 64, 2, 4),   # n = 2, even P: the two classes share no window
    ("n6_p2", 9, 9, 128, 6, 32, 2, 4),
    ("n4_c96", 8, 8, 256, 4, 96, 2, 2),          # c_out 96: one 96-wide channel block
])
def test_k3_class_pair_tiles(monkeypatch, cp, name, h, w, ci, n, co, pad, b):
    """K3p (both column parities per tile, bf16x2 stores) and the per-class K3 agree with the oracle."""
    import torch
    monkeypatch.setenv("SEGB200_IGEMM_GENERIC", "1")
    monkeypatch.setenv("SEGB200_K3_CP", cp)
    x, bank = _inputs(h, w, ci, n, co, b, 7000 + int(cp))
    layer = P.prepare_layer(bank, pad, compute="bf16")
    ref = O.forward_segregated_batch(x.float().cpu().numpy().astype(np.float64),
                                     O.bf16_round(bank).astype(np.float64), pad)
    y32 = layer.forward(x, path="igemm", out_dtype=torch.float32).cpu().numpy()
    rep = O.compare(y32, ref, 1e-4, 1e-5)
    assert rep["passed"], (name, cp, rep)
    yb = layer.forward(x, path="igemm").float().cpu().numpy()
    repb = O.compare(yb, ref, 2 ** -7, 1e-3 * float(np.abs(ref).max()))
    assert repb["passed"], (name, cp, repb)


# K3b's opt-in variants, kept working: M=256 CTA pairs for 128-wide rows (SEGB200_ROWS_PAIR=4)
# and K3's N tile forced to 128 run the default per-class accumulation order, so they must equal
# the default kernel bitwise; half-tile TMEM buffers (SEGB200_ROWS_HALF=1) and the unpaired M=64
# row split (SEGB200_ROWS_PAIR=0) accumulate each class's windows in another order, so they are
# held to the fp32 / bf16 output gates against the default instead
@pytest.mark.parametrize("env,val,shape,bitwise", [
    ("SEGB200_ROWS_PAIR", "4", (128, 128, 64, 4, 64, 2, 2), True),
    ("SEGB200_ROWS_HALF", "1", (128, 128, 64, 4, 64, 2, 2), False),
    ("SEGB200_ROWS_HALF", "1", (64, 128, 128, 4, 32, 2, 1), False),   # 2 channel blocks, odd batch
    ("SEGB200_ROWS_PAIR", "0", (64, 64, 128, 4, 64, 2, 2), False),   # M=64 row split: other order
    # (the default here is a 32-wide N tile for this small batch; another N tile width changes the
    # MMA's accumulation bits, measured)
    ("SEGB200_K3_NTILE", "128", (8, 8, 256, 4, 512, 2, 4), False),
])
def test_opt_in_variants(monkeypatch, env, val, shape, bitwise):
    import torch
    h, w, ci, n, co, pad, b = shape
    x, bank = _inputs(h, w, ci, n, co, b, 31 + h + co)
    layer = P.prepare_layer(bank, pad, compute="bf16")
    want = layer.forward(x, path="igemm")
    want32 = layer.forward(x, path="igemm", out_dtype=torch.float32)
    monkeypatch.setenv(env, val)
    got = layer.forward(x, path="igemm")
    got32 = layer.forward(x, path="igemm", out_dtype=torch.float32)
    torch.cuda.synchronize()
    if bitwise:
        assert torch.equal(got.view(torch.int16), want.view(torch.int16)), (env, val, shape)
    else:
        ref = want32.cpu().numpy().astype(np.float64)
        assert O.compare(got32.cpu().numpy(), ref, 1e-5, 1e-6)["passed"], (env, val, shape)
        assert O.compare(got.float().cpu().numpy(), ref, 2 ** -7, 1e-3 * float(np.abs(ref).max()))["passed"]


@pytest.mark.parametrize("xs,ws", [(1e-6, 1.0), (1.0, 1e-4), (3e4, 1.0), (1e6, 1e3), (2.0 ** -60, 2.0 ** 40)])
def test_3xfp16_scales_follow_magnitudes(xs, ws):
    """3xFP16 scales each operand by a power of two from its own maximum, so inputs far outside
    fp16's range (tiny, huge) keep the reference's fp32 gate (relative to the output scale)."""
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    b, ci, h, w, n, co, pad = 2, 128, 16, 16, 4, 64, 2
    x = device_unit_floats((b, ci, h, w), 31, dtype=torch.float32) * xs
    bank = (O.gen_kernel_bank(ci, co, n, 32) * ws).astype(np.float32)
    layer = P.prepare_layer(bank, pad)
    assert "3xFP16" in layer.describe_path(b, h, w)
    y = layer.forward(x).cpu().numpy()
    ref = O.forward_segregated_batch(x.cpu().numpy().astype(np.float64), bank.astype(np.float64), pad)
    scale = float(np.abs(ref).max())
    rep = O.compare(y, ref, 1e-5, 1e-6 * scale)
    assert rep["passed"], (xs, ws, rep)


def test_3xfp16_signed_data_error_bound():
    """signed N(0,1) data cancels: gate each element against 1e-5 x sum|x||w| (the
    conv of the magnitudes), the bound the reference's own fp32 engines meet on such data."""
    import torch
    b, ci, h, w, n, co, pad = 2, 256, 8, 8, 4, 128, 2
    rng = np.random.default_rng(5)
    xh = rng.standard_normal((b, ci, h, w)).astype(np.float32)
    bank = rng.standard_normal((ci, co, n, n)).astype(np.float32)
    layer = P.prepare_layer(bank, pad)
    assert "3xFP16" in layer.describe_path(b, h, w)
    y = layer.forward(torch.from_numpy(xh).cuda()).cpu().numpy().astype(np.float64)
    ref = O.forward_segregated_batch(xh.astype(np.float64), bank.astype(np.float64), pad)
    mag = O.forward_segregated_batch(np.abs(xh).astype(np.float64), np.abs(bank).astype(np.float64), pad)
    assert np.all(np.abs(y - ref) <= 1e-5 * mag + 1e-6), float((np.abs(y - ref) / mag).max())


def test_3xfp16_nan_propagates():
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    x = device_unit_floats((1, 64, 8, 8), 3, dtype=torch.float32)
    x[0, 5, 3, 4] = float("nan")
    layer = P.prepare_layer(O.gen_kernel_bank(64, 32, 4, 4), 2)
    assert "3xFP16" in layer.describe_path(1, 8, 8)
    y = layer.forward(x).cpu().numpy()
    ref = O.forward_segregated_batch(x.cpu().numpy().astype(np.float64), O.gen_kernel_bank(64, 32, 4, 4).astype(np.float64), 2)
    assert np.array_equal(np.isnan(y), np.isnan(ref))
    fin = ~np.isnan(ref)
    assert O.compare(y[fin], ref[fin], 1e-5, 1e-6)["passed"]


ROWS_F16_CASES = [  # K3b row-streaming 3xFP16 (fp32 in / out): 2-SM pairs over batch halves
    ("ebgan_l7_b2", 128, 128, 64, 4, 64, 2, 2),
    ("w64_b4", 32, 64, 64, 4, 64, 2, 4),
    ("c_out32", 16, 64, 64, 4, 32, 2, 2),
    ("h4_b2", 4, 64, 64, 4, 64, 2, 2),
    ("b6_h8", 8, 128, 64, 4, 64, 2, 6),
    ("ebgan_l6_b2", 64, 64, 128, 4, 64, 2, 2),   # two 64-channel passes, the second accumulating
    ("c_in96_c32", 16, 64, 96, 4, 32, 2, 4),     # a partial second channel block
]


@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b", ROWS_F16_CASES)
def test_rows_3xfp16_fp32_gate(monkeypatch, name, h, w, ci, n, co, pad, b):
    """fp32 layers on the row-streaming kernel (3xFP16) meet the reference's fp32 gate, and agree
    with the generic K3 3xFP16 kernel (SEGB200_IGEMM_GENERIC=1) to the same gate"""
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    x = device_unit_floats((b, ci, h, w), 700 + ci, dtype=torch.float32)
    bank = O.gen_kernel_bank(ci, co, n, 701 + ci)
    layer = P.prepare_layer(bank, pad)
    kern = layer.describe_path(b, h, w)
    assert "K3b" in kern and "3xFP16" in kern, (name, kern)
    y = layer.forward(x).cpu().numpy()
    ref = O.forward_segregated_batch(x.cpu().numpy().astype(np.float64), bank.astype(np.float64), pad)
    rep = O.compare(y, ref, 1e-5, 1e-6)
    assert rep["passed"], (name, rep)
    monkeypatch.setenv("SEGB200_IGEMM_GENERIC", "1")
    assert "K3 implicit GEMM (3xFP16)" in layer.describe_path(b, h, w)
    yg = layer.forward(x).cpu().numpy()
    assert O.compare(y, yg.astype(np.float64), 1e-5, 1e-6)["passed"], name


@pytest.mark.parametrize("compute", ["bf16", "fp32"])
@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b,ksplit", [
    ("dcgan_l2_b1", 4, 4, 1024, 4, 512, 2, 1, None),     # auto split K (tiles cannot cover the SMs)
    ("ebgan_l2_b1", 4, 4, 2048, 4, 1024, 2, 1, None),
    ("dcgan_l3_b2", 8, 8, 512, 4, 256, 2, 2, None),
    ("forced_k3", 8, 8, 256, 4, 128, 2, 4, "3"),         # an uneven split of 16 k-steps
    ("odd_pad_ks", 8, 8, 256, 2, 64, 1, 2, "2"),
])
def test_split_k_small_batches(monkeypatch, compute, name, h, w, ci, n, co, pad, b, ksplit):
    """split K (fp32 partials summed in a fixed order by a second kernel) matches the oracle at
    the path's gate and is bitwise reproducible"""
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    if ksplit:
        monkeypatch.setenv("SEGB200_K3_KSPLIT", ksplit)
    monkeypatch.setenv("SEGB200_K3_CP", "0")
    tdt = torch.bfloat16 if compute == "bf16" else torch.float32
    x = device_unit_floats((b, ci, h, w), 300 + ci, dtype=tdt)
    bank = O.gen_kernel_bank(ci, co, n, 301 + ci)
    layer = P.prepare_layer(bank, pad, compute=compute)
    y = layer.forward(x, path="igemm", out_dtype=torch.float32)
    assert torch.equal(y, layer.forward(x, path="igemm", out_dtype=torch.float32))
    xr = x.float().cpu().numpy().astype(np.float64)
    br = (O.bf16_round(bank) if compute == "bf16" else bank).astype(np.float64)
    ref = O.forward_segregated_batch(xr, br, pad)
    tol = (1e-4, 1e-5) if compute == "bf16" else (1e-5, 1e-6)
    rep = O.compare(y.cpu().numpy(), ref, *tol)
    assert rep["passed"], (name, compute, rep)


@pytest.mark.parametrize("compute", ["bf16", "fp32"])
@pytest.mark.parametrize("name,h,w,ci,n,co,pad,b,noswap", [
    ("dcgan_l2_b1", 4, 4, 1024, 4, 512, 2, 1, False),
    ("dcgan_l3_b1", 8, 8, 512, 4, 256, 2, 1, False),
    ("ebgan_l2_b2", 4, 4, 2048, 4, 1024, 2, 2, False),
    ("odd_pad_b3", 4, 4, 256, 2, 128, 1, 3, False),   # class grid 4x4 (P=1, n=2) x 3 samples: 48 positions
    ("dcgan_l2_b1_unswapped", 4, 4, 1024, 4, 512, 2, 1, True),
])
def test_swapped_operands_tiny_batches(monkeypatch, compute, name, h, w, ci, n, co, pad, b, noswap):
    """the opt-in swapped-operand K3 (SEGB200_K3_SWAP=1: weights as the MMA's M side, the class
    positions as N, PM 3) with split K computes the same layer as the default layout"""
    import torch
    from paper_2502_20493_b200.synth import device_unit_floats
    if not noswap:
        monkeypatch.setenv("SEGB200_K3_SWAP", "1")
    tdt = torch.bfloat16 if compute == "bf16" else torch.float32
    x = device_unit_floats((b, ci, h, w), 500 + ci, dtype=tdt)
    bank = O.gen_kernel_bank(ci, co, n, 501 + ci)
    layer = P.prepare_layer(bank, pad, compute=compute)
    kern = layer.describe_path(b, h, w)
    assert ("swapped" in kern) != noswap, kern
    y = layer.forward(x, out_dtype=torch.float32)
    assert torch.equal(y, layer.forward(x, out_dtype=torch.float32))
    xr = x.float().cpu().numpy().astype(np.float64)
    br = (O.bf16_round(bank) if compute == "bf16" else bank).astype(np.float64)
    ref = O.forward_segregated_batch(xr, br, pad)
    tol = (1e-4, 1e-5) if compute == "bf16" else (1e-5, 1e-6)
    rep = O.compare(y.cpu().numpy(), ref, *tol)
    assert rep["passed"], (name, compute, kern, rep)
