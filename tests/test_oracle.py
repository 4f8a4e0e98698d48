"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from /root/reference). CPU only."""

import numpy as np
import pytest

from oracle import c_forward_f64
from oracle import segconv_oracle as O
from tests.conftest import golden_cases


def test_known_answers(golden):
    x = np.array([[[1, 2], [3, 4]]], dtype=np.float32)
    k = np.array([[[[1, 2], [3, 4]]]], dtype=np.float32)
    np.testing.assert_array_equal(O.forward_segregated(x, k, 0)[0], golden["kat_p0"])
    np.testing.assert_array_equal(O.forward_segregated(x, k, 1)[0], golden["kat_p1"])
    np.testing.assert_array_equal(golden["kat_p1"],
                                  [[4, 3, 8, 6], [2, 1, 4, 2], [12, 9, 16, 12], [6, 3, 8, 4]])
    np.testing.assert_array_equal(O.forward_reference(x, k, 1)[0], golden["kat_p1_ref"])
    ones = np.ones((1, 1, 2, 2), np.float32)
    np.testing.assert_array_equal(O.forward_segregated(x, ones, 0)[0], golden["kat_ones"])


def test_splitmix_and_streams(golden):
    for s_in, s_out in zip(golden["splitmix_in"], golden["splitmix_out"]):
        assert O.splitmix64(int(s_in)) == int(s_out)
    assert O.splitmix64(42) == 0xBDD732262FEB6E95
    for s, row in zip(golden["unit_floats_seeds"], golden["unit_floats"]):
        assert np.array_equal(O.unit_floats(64, int(s)).view(np.uint32), row.view(np.uint32))
    assert np.array_equal(O.gen_synthetic(3, 5, 7, 9), golden["gen_synthetic_3_5_7_s9"])
    assert np.array_equal(O.gen_kernel_bank(2, 3, 4, 11), golden["gen_kernel_bank_2_3_4_s11"])


def test_mult_counts(golden):
    for spec, seg in zip(golden["count_specs"], golden["count_seg"]):
        h, w, n, p, ci, co = (int(v) for v in spec)
        assert O.mult_count_segregated(h, w, n, p, ci, co) == int(seg)
    assert O.mult_count_segregated(4, 4, 5, 0) == 64


def test_c_oracle_counts(golden):
    from oracle import c_oracle
    lib = c_oracle()
    for spec, seg in zip(golden["count_specs"], golden["count_seg"]):
        h, w, n, p, ci, co = (int(v) for v in spec)
        assert lib.oracle_mult_count(h, w, n, p, ci, co) == int(seg)


def test_segregation(golden):
    for n in range(2, 10):
        kk = np.arange(n * n, dtype=np.float32).reshape(n, n)
        subs = O.segregate(kk)
        for sub, name in zip(subs, ("k00", "k01", "k10", "k11")):
            assert np.array_equal(sub, golden[f"seg_n{n}_{name}"])
        assert np.array_equal(O.merge(subs, n).view(np.uint32), kk.view(np.uint32))


def test_numpy_oracle_matches_reference_cases(golden):
    for i, x, bank, pad, seg32, seg64, ref64 in golden_cases(golden):
        got64 = O.forward_segregated(x, bank, pad)
        assert got64.shape == seg64.shape
        assert np.max(np.abs(got64 - seg64)) < 1e-12, i
        assert np.max(np.abs(got64 - ref64)) < 1e-12, i
        got32 = O.forward_segregated(x.astype(np.float32), bank.astype(np.float32), pad)
        assert got32.dtype == np.float32
        assert O.compare(got32, seg32, 1e-6, 1e-7)["passed"], i


def test_c_oracle_matches_reference_cases(golden):
    for i, x, bank, pad, seg32, seg64, ref64 in golden_cases(golden):
        got = c_forward_f64(x[None], bank, pad)[0]
        assert np.max(np.abs(got - seg64)) < 1e-12, i


def test_scalar_oracle_counts_and_values(golden):
    # engines.py:379-406 literal form: counts and write-once
    for i, x, bank, pad, seg32, seg64, ref64 in list(golden_cases(golden))[:25]:
        out, mults, writes = O.forward_scalar(x, bank, pad)
        assert writes == out.size
        c_in, h, w = x.shape
        n = bank.shape[2]
        assert mults == O.mult_count_segregated(h, w, n, pad, c_in, bank.shape[1])
        assert np.max(np.abs(out - seg64)) < 1e-12


def test_gan_shaped_layers(golden):
    for i in range(int(golden["n_gan"])):
        h, w, ci, n, co, pad, in_seed, bank_seed = (int(v) for v in golden[f"gan{i}_meta"])
        x = O.gen_synthetic(ci, h, w, in_seed)
        bank = O.gen_kernel_bank(ci, co, n, bank_seed)
        got = O.forward_segregated(x, bank, pad)
        assert O.compare(got, golden[f"gan{i}_out"], 1e-5, 1e-6)["passed"], i


def test_batched_sample_equals_per_sample_seed():
    # batch stream sample j == gen_synthetic(C,H,W, seed + j*C*H*W)
    c, h, w, b, seed = 2, 3, 5, 4, 99
    stream = O.unit_floats(b * c * h * w, seed).reshape(b, c, h, w)
    for j in range(b):
        assert np.array_equal(stream[j], O.gen_synthetic(c, h, w, seed + j * c * h * w))


@pytest.mark.parametrize("pad", [0, 1, 2, 3])
def test_compare_semantics(pad):
    a = np.array([1.0, 2.0])
    b = np.array([1.0, 2.0 + 1e-3])
    assert not O.compare(a, b)["passed"]
    assert O.compare(a, b, 1e-2, 1e-6)["passed"]
    assert not O.compare(np.zeros((2, 2)), np.zeros((3, 3)))["shapes_match"]


def test_counted_engines(golden):
    """the scalar restatements (engines.py:353-406) reproduce the reference's counted engines
    bit for bit, counters included"""
    for i in range(int(golden["n_cnt"])):
        m, k, pad = golden[f"cnt{i}_map"], golden[f"cnt{i}_kernel"], int(golden[f"cnt{i}_pad"])
        c = golden[f"cnt{i}_counts"]
        ref, rm, rw = O.forward_scalar_reference(m, k, pad)
        seg, sm, sw = O.forward_scalar(m[None], k[None, None], pad)
        assert np.array_equal(ref, golden[f"cnt{i}_ref"]), i
        assert np.array_equal(seg[0], golden[f"cnt{i}_seg"]), i
        assert (rm, rw, sm, sw) == tuple(int(v) for v in c), i
