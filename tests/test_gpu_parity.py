"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
outputs and the pinned CPU oracle. Mirrors the reference's own suites
(tests/test_engines.py, tests/test_acceptance.py, tests/test_segregation.py).

Tolerances: fp32 rel 1e-5 / abs 1e-6 and fp64 abs 1e-12 (the reference's,
test_acceptance.py:31-32); bf16 gates are stated in test_bf16_*."""

import numpy as np
import pytest

import paper_2502_20493_b200 as P
from oracle import segconv_oracle as O
from tests.conftest import golden_cases

pytestmark = pytest.mark.gpu
F32 = np.float32
REL32, ABS32, ABS64 = 1e-5, 1e-6, 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _ok32(a, b):
    return a.shape == b.shape and bool(np.all(np.abs(a.astype(np.float64) - b) <= ABS32 + REL32 * np.abs(b)))


# --- frozen known answers (test_engines.py:65-107) ---------------------------------------

def test_known_answers(golden):
    x = np.array([[1, 2], [3, 4]], dtype=F32)
    k = np.array([[1, 2], [3, 4]], dtype=F32)
    np.testing.assert_array_equal(P.transpose_conv_segregated(x, P.segregate_kernel(k), 0), golden["kat_p0"])
    np.testing.assert_array_equal(P.transpose_conv_segregated(x, P.segregate_kernel(k), 1), golden["kat_p1"])
    np.testing.assert_array_equal(P.transpose_conv_reference(x, k, 1), golden["kat_p1_ref"])
    np.testing.assert_array_equal(
        P.transpose_conv_segregated(x, P.segregate_kernel(np.ones((2, 2), F32)), 0), x)
    out = P.transpose_conv_segregated(np.ones((4, 4), F32), P.segregate_kernel(np.ones((5, 5), F32)), 2)
    assert out.shape == (7, 7)


def test_inconsistent_subkernels_rejected():
    with pytest.raises(P.SpecError):
        subs = P.segregate_kernel(np.ones((9, 9), F32))
        P.transpose_conv_segregated(np.ones((1, 1), F32), subs, 0)
    subs = P.segregate_kernel(np.ones((3, 3), F32))
    broken = type(subs)(size=3, k00=subs.k00, k01=subs.k01, k10=subs.k10, k11=np.zeros((2, 2), F32))
    with pytest.raises(P.ShapeError):
        P.transpose_conv_segregated(np.ones((4, 4), F32), broken, 0)


# --- K1: device segregation (test_segregation.py, acceptance criterion 3) ----------------

def test_device_segregation_matches_reference(golden):
    for n in range(2, 10):
        kk = np.arange(n * n, dtype=F32).reshape(n, n)
        subs = P.segregate_kernel(kk)
        for name in ("k00", "k01", "k10", "k11"):
            np.testing.assert_array_equal(getattr(subs, name), golden[f"seg_n{n}_{name}"])
        assert subs.element_count() == n * n
        rng = np.random.default_rng(n)
        for dt in (np.float32, np.float64):
            k = rng.random((n, n)).astype(dt)
            back = P.merge_subkernels(P.segregate_kernel(k))
            assert back.dtype == dt and np.array_equal(back.view(np.uint8), k.view(np.uint8))
    five = P.segregate_kernel(np.ones((5, 5), F32))
    assert (five.k00.size, five.k01.size, five.k10.size, five.k11.size) == (9, 6, 6, 4)


# --- reference golden cases (random layers, fp32 and fp64) --------------------------------

def test_golden_cases_fp32_fp64(golden):
    for i, x, bank, pad, seg32, seg64, ref64 in golden_cases(golden):
        got32 = P.layer_forward(x.astype(F32), bank.astype(F32), pad)
        assert got32.dtype == np.float32
        assert _ok32(got32, seg32.astype(np.float64)), i
        got64 = P.layer_forward(x, bank, pad)
        assert got64.dtype == np.float64
        assert float(np.max(np.abs(got64 - seg64))) < ABS64, i
        assert float(np.max(np.abs(got64 - ref64))) < ABS64, i


def test_gan_shaped_golden(golden):
    for i in range(int(golden["n_gan"])):
        h, w, ci, n, co, pad, in_seed, bank_seed = (int(v) for v in golden[f"gan{i}_meta"])
        x = O.gen_synthetic(ci, h, w, in_seed)
        bank = O.gen_kernel_bank(ci, co, n, bank_seed)
        got = P.layer_forward(x, bank, pad)
        assert P.compare_outputs(got, golden[f"gan{i}_out"]).passed, i


# --- acceptance criterion 1: 1000-case oracle equivalence (test_acceptance.py:53-82) -------

def _draw_case(rng):
    while True:
        in_h = int(rng.integers(1, 33))
        in_w = int(rng.integers(1, 33))
        n = int(rng.integers(2, 10))
        pad = int(rng.integers(0, 5))
        if 2 * in_h + 2 * pad - n >= 1 and 2 * in_w + 2 * pad - n >= 1:
            return in_h, in_w, n, pad, int(rng.integers(1, 5)), int(rng.integers(1, 5))


def test_acceptance_1_oracle_equivalence():
    rng = np.random.default_rng(20260810)
    pads = {p: 0 for p in range(5)}
    worst32 = worst64 = 0.0
    for _ in range(1000):
        h, w, n, pad, ci, co = _draw_case(rng)
        pads[pad] += 1
        x64 = rng.random((ci, h, w))
        b64 = rng.random((ci, co, n, n))
        ref64 = O.forward_segregated(x64, b64, pad)  # oracle, fp64
        seg32 = P.layer_forward(x64.astype(F32), b64.astype(F32), pad)
        assert _ok32(seg32, ref64), (h, w, n, pad, ci, co)
        worst32 = max(worst32, float(np.max(np.abs(seg32 - ref64))))
        seg64 = P.layer_forward(x64, b64, pad)
        d64 = float(np.max(np.abs(seg64 - ref64)))
        assert d64 <= ABS64, (h, w, n, pad, ci, co, d64)
        worst64 = max(worst64, d64)
    assert all(v > 0 for v in pads.values())
    print(f"ACCEPTANCE 1 (GPU): worst fp32 abs {worst32:.2e}, worst fp64 abs {worst64:.2e}")


# --- acceptance 2: odd padding swap (test_acceptance.py:85-105) ---------------------------

def test_acceptance_2_odd_padding_swap():
    rng = np.random.default_rng(20260811)
    checked = 0
    for pad in (1, 3):
        for n in range(2, 10):
            for h in (1, 2, 3, 5, 8):
                if 2 * h + 2 * pad - n < 1:
                    continue
                x = rng.random((h, h + 1)).astype(F32)
                k = rng.random((n, n)).astype(F32)
                ref = O.forward_reference(x[None].astype(np.float64), k[None, None].astype(np.float64), pad)[0]
                seg = P.transpose_conv_segregated(x, P.segregate_kernel(k), pad)
                assert _ok32(seg, ref), (pad, n, h)
                checked += 1
    assert checked >= 60


# --- acceptance 4 / write-once: every element written, nothing outside written ------------

@pytest.mark.parametrize("h,n,pad", [(4, 5, 0), (4, 4, 2), (3, 3, 1), (5, 7, 2), (2, 2, 0), (6, 5, 3),
                                     (1, 2, 1), (28, 3, 1), (9, 9, 4)])
def test_acceptance_4_exact_coverage(h, n, pad):
    import torch
    rng = np.random.default_rng(h * 100 + n * 10 + pad)
    ci, co, b = 2, 3, 3
    x = rng.random((b, ci, h, h + 1)).astype(F32)
    bank = rng.random((ci, co, n, n)).astype(F32)
    layer = P.prepare_layer(bank, pad)
    oh, ow = layer.output_shape(h, h + 1)
    total = b * co * oh * ow
    guard = 4096
    buf = torch.full((guard + total + guard,), float("nan"), device="cuda")
    sentinel = buf.clone()
    y = buf[guard:guard + total].view(b, co, oh, ow)
    layer.forward(torch.from_numpy(x).cuda(), out=y)
    torch.cuda.synchronize()
    assert not torch.isnan(y).any()  # every output element written
    assert torch.isnan(buf[:guard]).all() and torch.isnan(buf[guard + total:]).all()  # nothing else
    del sentinel
    ref = np.stack([O.forward_segregated(xi.astype(np.float64), bank.astype(np.float64), pad) for xi in x])
    assert _ok32(y.cpu().numpy(), ref)


def test_nan_input_reaches_every_output():
    # test_engines.py:235-247
    rng = np.random.default_rng(2)
    for pad in (0, 1):
        for n in (2, 3, 4, 5):
            nh = int(rng.integers(2, 7))
            if 2 * nh + 2 * pad - n < 1:
                continue
            out = P.layer_forward(np.full((1, nh, nh), np.nan, F32), np.ones((1, 1, n, n), F32), pad)
            assert np.isnan(out).all(), (nh, n, pad)


def test_delta_kernel_scatter_exact():
    rng = np.random.default_rng(5)
    x = rng.random((5, 6)).astype(F32)
    for n in (2, 3, 4, 5):
        k = np.zeros((n, n), F32)
        k[0, 0] = 1.0
        seg = P.transpose_conv_segregated(x, P.segregate_kernel(k), 0)
        for i in range(seg.shape[0]):
            for j in range(seg.shape[1]):
                want = x[i // 2, j // 2] if i % 2 == 0 and j % 2 == 0 else 0.0
                assert seg[i, j] == want


def test_linearity_in_input():
    rng = np.random.default_rng(9)
    a = rng.random((4, 5)).astype(F32)
    b = rng.random((4, 5)).astype(F32)
    subs = P.segregate_kernel(rng.random((3, 3)).astype(F32))
    f = lambda m: P.transpose_conv_segregated(m, subs, 1)  # noqa: E731
    np.testing.assert_allclose(f(2.0 * a + 0.5 * b), 2.0 * f(a) + 0.5 * f(b), rtol=1e-5, atol=1e-6)


def test_layer_semantics():
    rng = np.random.default_rng(12)
    x = rng.random((3, 4, 4))
    bank = rng.random((3, 2, 3, 3))
    out = P.layer_forward(x, bank, 1)
    manual = np.zeros_like(out)
    for co in range(2):
        for ci in range(3):
            manual[co] += O.forward_reference(x[ci:ci + 1], bank[ci:ci + 1, co:co + 1], 1)[0]
    np.testing.assert_allclose(out, manual, rtol=1e-12, atol=1e-12)
    assert P.layer_forward(np.zeros((1024, 4, 4), F32), np.zeros((1024, 512, 4, 4), F32), 2).shape == (512, 8, 8)
    with pytest.raises(P.ShapeError):
        P.layer_forward(np.ones((2, 4, 4), F32), np.ones((3, 1, 3, 3), F32), 1)
    with pytest.raises(ValueError):
        P.layer_forward(np.ones((1, 4, 4), F32), np.ones((1, 1, 2, 2), F32), 0, threads=0)


def test_reference_engine_on_gpu():
    rng = np.random.default_rng(33)
    for nh, n, pad in [(4, 3, 0), (5, 4, 2), (3, 5, 2), (6, 3, 1), (4, 7, 4)]:
        x = rng.random((2, nh, nh + 2))
        k = rng.random((2, 3, n, n))
        got = P.layer_forward(x, k, pad, engine=P.ENGINE_REFERENCE)
        want = O.forward_reference(x, k, pad)
        assert float(np.max(np.abs(got - want))) < 1e-12


# --- determinism (test_engines.py:302-330, acceptance 8) ----------------------------------

def test_determinism_bitwise():
    rng = np.random.default_rng(21)
    x = rng.random((6, 9, 8)).astype(F32)
    bank = rng.random((6, 40, 5, 5)).astype(F32)
    a = P.layer_forward(x, bank, 2, threads=2)
    b = P.layer_forward(x, bank, 2, threads=2)
    c = P.layer_forward(x, bank, 2, threads=1)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(a.view(np.uint32), c.view(np.uint32))
    layer = P.prepare_layer(bank, 2)
    assert np.array_equal(layer.forward(x), a) and np.array_equal(layer.forward(x), a)


def test_batched_equals_per_sample():
    import torch
    rng = np.random.default_rng(4)
    x = rng.random((5, 3, 11, 7)).astype(F32)
    bank = rng.random((3, 4, 5, 5)).astype(F32)
    layer = P.prepare_layer(bank, 3)
    yb = layer.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    for j in range(5):
        assert np.array_equal(yb[j].view(np.uint32), layer.forward(x[j]).view(np.uint32))


# --- large shapes: BASELINE configs vs the oracle -----------------------------------------

@pytest.mark.parametrize("name,h,ci,n,co,pad,b", [
    ("mnist_p0", 28, 1, 3, 1, 0, 64), ("mnist_p1", 28, 1, 3, 1, 1, 64), ("mnist_p2", 28, 1, 3, 1, 2, 64),
    ("ds224_k3", 224, 3, 3, 1, 2, 2), ("ds224_k4", 224, 3, 4, 1, 1, 2), ("ds512_k5", 512, 3, 5, 3, 2, 1),
    ("ds64_k5_c2", 64, 2, 5, 3, 1, 4), ("dcgan_l5", 32, 128, 4, 3, 2, 2), ("ebgan_l7", 128, 64, 4, 64, 2, 1),
    ("dcgan_l2", 4, 1024, 4, 512, 2, 2)])
def test_baseline_configs_fp32(name, h, ci, n, co, pad, b):
    import torch
    in_seed, bank_seed = O.harness_seeds(0, 0)
    x = O.unit_floats(b * ci * h * h, in_seed).reshape(b, ci, h, h)
    bank = O.gen_kernel_bank(ci, co, n, bank_seed)
    y = P.prepare_layer(bank, pad).forward(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = O.forward_segregated_batch(x.astype(np.float64), bank.astype(np.float64), pad)
    rep = O.compare(y, ref, REL32, ABS32)
    assert rep["passed"], (name, rep)


def test_device_synth_bits_match_reference():
    from paper_2502_20493_b200.synth import device_unit_floats
    import torch
    for seed in (0, 42, 2**63, (1 << 64) - 1, 123456789):
        got = device_unit_floats((4097,), seed).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), O.unit_floats(4097, seed).view(np.uint32))
    got = device_unit_floats((3, 2, 5), 9, dtype=torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(got, O.bf16_round(O.unit_floats(30, 9)).reshape(3, 2, 5))


def test_torch_conv_transpose_cross_check():
    # test_engines.py:354-369 mapping: conv_transpose2d(x, flip(K), stride 2, padding n-1-P)
    import torch
    rng = np.random.default_rng(3)
    for h, n, pad, ci, co in [(16, 4, 2, 8, 16), (9, 5, 3, 3, 2), (12, 3, 1, 4, 4)]:
        x = torch.from_numpy(rng.random((2, ci, h, h))).cuda()
        k = torch.from_numpy(rng.random((ci, co, n, n))).cuda()
        ours = P.prepare_layer(k, pad).forward(x)
        theirs = torch.nn.functional.conv_transpose2d(x, k.flip(2, 3), stride=2, padding=n - 1 - pad)
        assert float((ours - theirs).abs().max()) < 1e-12


@pytest.mark.parametrize("compute,shape", [("fp32", (9, 3, 17, 13, 5, 2, 4)), ("bf16", (10, 128, 16, 16, 4, 2, 64)),
                                           ("bf16", (6, 64, 128, 128, 4, 2, 64))])
def test_batch_sharding_bitwise(compute, shape):
    """Each rank's shard (parallel.shard_range) reproduces its slice of the 1-GPU output bit
    for bit, for the direct, K3 and K3b paths: no collective is needed on the hot path."""
    import torch
    from paper_2502_20493_b200.parallel import shard_batch
    from paper_2502_20493_b200.synth import device_unit_floats
    b, ci, h, w, n, pad, co = shape
    dt = torch.bfloat16 if compute == "bf16" else torch.float32
    x = device_unit_floats((b, ci, h, w), 3, dtype=dt)
    bank = O.gen_kernel_bank(ci, co, n, 4)
    layer = P.prepare_layer(bank, pad, compute=compute)
    full = layer.forward(x)
    for world in (2, 3, 4):
        parts = [layer.forward(shard_batch(x, world, r).contiguous()) for r in range(world)]
        joined = torch.cat(parts)
        assert torch.equal(joined.view(torch.int16 if dt == torch.bfloat16 else torch.int32),
                           full.view(torch.int16 if dt == torch.bfloat16 else torch.int32))


@pytest.mark.parametrize("compute,tdt,b,h", [("bf16", "bfloat16", 16, 64), ("bf16", "bfloat16", 7, 128),
                                              ("fp32", "float32", 5, 128)])
def test_host_pipeline_bitwise_equals_device_call(compute, tdt, b, h):
    """Host batches >= 8 MB go through the chunked H2D / compute / D2H pipeline; the result is
    bitwise that of one device-resident call, with and without out=, pinned or pageable."""
    import torch
    dt = getattr(torch, tdt)
    w = h
    ci, co, n, pad = 64, 64, 4, 2
    bank = O.gen_kernel_bank(ci, co, n, 3)
    layer = P.prepare_layer(bank, pad, compute=compute)
    g = torch.Generator().manual_seed(b)
    xh = torch.rand((b, ci, h, w), generator=g).to(dt)
    assert xh.numel() * xh.element_size() >= 8 << 20  # takes the pipelined path
    ref = layer.forward(xh.cuda()).cpu()
    y1 = layer.forward(xh.pin_memory())
    assert y1.device.type == "cpu" and torch.equal(y1, ref)
    out = torch.empty_like(ref).pin_memory()
    y2 = layer.forward(xh.pin_memory(), out=out)
    torch.cuda.synchronize()
    assert y2 is out and torch.equal(out, ref)
    y3 = layer.forward(xh)  # pageable input
    assert torch.equal(y3, ref)
