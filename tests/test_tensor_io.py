"""Dataset-input formats: the host decode mirrors the reference's
tensor_io.py (header rules, FormatError messages, bit patterns -- the reference's own
tests/test_tensor_io.py cases restated), and the device loaders are bitwise the host decode.
"""

import struct

import numpy as np
import pytest

from oracle import segconv_oracle as O
from paper_2502_20493_b200 import tensor_io as T


def ppm_bytes(width, height, pixels, magic=b"P6"):
    return magic + b" %d %d 255\n" % (width, height) + bytes(pixels)


def test_ppm_decode_matches_reference_formula():
    rng = np.random.default_rng(3)
    px = rng.integers(0, 256, size=5 * 7 * 3, dtype=np.uint8)
    t = T.parse_ppm(ppm_bytes(7, 5, px))
    want = px.reshape(5, 7, 3).transpose(2, 0, 1).astype(np.float32) / np.float32(255.0)  # tensor_io.py:52
    assert t.shape == (3, 5, 7) and t.dtype == np.float32
    assert np.array_equal(t.view(np.uint32), want.view(np.uint32))


def test_ppm_known_answers():
    assert np.array_equal(T.parse_ppm(ppm_bytes(1, 1, [255, 0, 0]))[:, 0, 0], [1.0, 0.0, 0.0])
    t = T.parse_ppm(ppm_bytes(2, 1, [10, 20, 30, 40, 50, 60]))  # channel deinterleave
    np.testing.assert_allclose(t[:, 0, 1] * 255.0, [40, 50, 60])
    assert T.parse_ppm(b"P6\n# c\n2 # inline\n1\n255\n" + bytes(6)).shape == (3, 1, 2)


@pytest.mark.parametrize("data,match", [
    (ppm_bytes(1, 1, [0, 0, 0], magic=b"P5"), "P6"),
    (b"P6 1 1 65535\n" + bytes(6), "maxval"),
    (ppm_bytes(2, 2, [0] * 5), "truncated"),
    (b"P6 one 1 255\n" + bytes(3), "non-numeric"),
    (b"P6 0 1 255\n", "size"),
    (b"P6 1 1 255", "whitespace|end of data"),
])
def test_ppm_errors(data, match):
    with pytest.raises(T.FormatError, match=match):
        T.parse_ppm(data)


def test_sct_roundtrip_and_layout(tmp_path):
    t = O.gen_synthetic(3, 7, 5, 4)
    p = tmp_path / "t.sct"
    T.save_raw_tensor(t, p)
    back = T.load_raw_tensor(p)
    assert np.array_equal(back.view(np.uint32), t.view(np.uint32))
    blob = T.tensor_to_sct_bytes(np.arange(8, dtype=np.float32).reshape(2, 2, 2))
    assert blob[:4] == b"SCT1" and struct.unpack("<III", blob[4:16]) == (2, 2, 2)
    assert list(struct.unpack("<8f", blob[16:])) == list(range(8))


@pytest.mark.parametrize("data,match", [
    (b"NOPE" + bytes(16), "magic"),
    (b"SCT1\x01", "too short"),
    (b"SCT1" + struct.pack("<III", 0, 2, 2), "dims"),
    (b"SCT1" + struct.pack("<III", 1, 2, 2) + bytes(12), "mismatch"),
    (b"SCT1" + struct.pack("<III", 1, 1, 1) + bytes(5), "mismatch"),
])
def test_sct_errors(data, match):
    with pytest.raises(T.FormatError, match=match):
        T.sct_bytes_to_tensor(data)


def test_format_error_is_value_error():
    assert issubclass(T.FormatError, ValueError)


# ------------------------------------------------------------------ device loaders

@pytest.mark.gpu
def test_ppm_batch_on_device_bitwise():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rng = np.random.default_rng(11)
    imgs = [ppm_bytes(33, 17, rng.integers(0, 256, size=33 * 17 * 3, dtype=np.uint8)) for _ in range(3)]
    d = T.load_ppm_batch(imgs)
    want = np.stack([T.parse_ppm(b) for b in imgs])
    assert d.shape == (3, 3, 17, 33) and d.dtype == torch.float32
    assert np.array_equal(d.cpu().numpy().view(np.uint32), want.view(np.uint32))
    one = T.ppm_to_device(imgs[1], dtype=torch.bfloat16)
    assert torch.equal(one.cpu(), torch.from_numpy(want[1]).to(torch.bfloat16))
    with pytest.raises(T.FormatError):
        T.load_ppm_batch([imgs[0], ppm_bytes(2, 2, [0] * 12)])


@pytest.mark.gpu
def test_dataset_image_through_layer(tmp_path):
    """paper 4.1 path: a PPM image straight to the device, one segregated layer, vs the oracle"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2502_20493_b200 as P
    rng = np.random.default_rng(5)
    path = tmp_path / "img.ppm"
    path.write_bytes(ppm_bytes(40, 24, rng.integers(0, 256, size=40 * 24 * 3, dtype=np.uint8)))
    sct = tmp_path / "img.sct"
    T.save_raw_tensor(T.load_ppm(path), sct)
    bank = O.gen_kernel_bank(3, 1, 5, 9)
    layer = P.prepare_layer(bank, 2)
    y = layer.forward(T.ppm_to_device(path))
    ref = O.forward_segregated(T.load_ppm(path).astype(np.float64), bank.astype(np.float64), 2)
    assert O.compare(y.cpu().numpy(), ref, 1e-5, 1e-6)["passed"]
    assert torch.equal(T.sct_to_device(sct), T.ppm_to_device(path))
