"""Dataset images to the device (paper_2502_20493_b200/tensor_io.py).

The decoded values are pinned to the reference's own decode: its parse_ppm from the unmodified
package in baseline/_ref when installed, else the formula it implements (tensor_io.py:52:
pixels.transpose(2, 0, 1).astype(float32) / float32(255)). The fused path (the u8 payload decoded
inside the direct kernel's loads) must equal the layer on the decoded batch bit for bit.
"""

import os
import struct
import sys

import numpy as np
import pytest

from oracle import segconv_oracle as O
from paper_2502_20493_b200 import tensor_io as T
from tests.conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")


def ppm_bytes(width, height, pixels, magic=b"P6", sep=b" "):
    return magic + sep + b"%d%s%d%s255\n" % (width, sep, height, sep) + bytes(pixels)


def reference_decode(data: bytes) -> np.ndarray:
    if os.path.isdir(os.path.join(REF, "segconv")):
        if REF not in sys.path:
            sys.path.insert(0, REF)
        from segconv.tensor_io import parse_ppm
        return parse_ppm(data)
    h, w, off = T.ppm_geometry(data)
    px = np.frombuffer(data, dtype=np.uint8, count=h * w * 3, offset=off).reshape(h, w, 3)
    return px.transpose(2, 0, 1).astype(np.float32) / np.float32(255.0)


def test_geometry_of_headers():
    assert T.ppm_geometry(ppm_bytes(7, 5, bytes(105))) == (5, 7, len(b"P6 7 5 255\n"))
    data = b"P6\n# a comment\n2 # inline\n1\n255\n" + bytes(6)
    h, w, off = T.ppm_geometry(data)
    assert (h, w) == (1, 2) and data[off:] == bytes(6)
    data = b"P6\t3\r\n2\x0b255 " + bytes(range(18))
    h, w, off = T.ppm_geometry(data)
    assert (h, w) == (2, 3) and data[off:off + 18] == bytes(range(18))


@pytest.mark.parametrize("data,match", [
    (ppm_bytes(1, 1, [0, 0, 0], magic=b"P5"), "P6"),
    (b"P6 1 1 65535\n" + bytes(6), "maxval"),
    (ppm_bytes(2, 2, [0] * 5), "truncated"),
    (b"P6 one 1 255\n" + bytes(3), "non-numeric"),
    (b"P6 0 1 255\n", "size"),
    (b"P6 1 1 255", "malformed"),
])
def test_ppm_errors(data, match):
    with pytest.raises(T.FormatError, match=match):
        T.ppm_geometry(data)


def test_format_error_is_value_error():
    assert issubclass(T.FormatError, ValueError)


def test_reference_decode_agrees_on_comments():
    """the header scan locates the same payload the reference's tokenizer does"""
    rng = np.random.default_rng(2)
    px = rng.integers(0, 256, size=4 * 3 * 3, dtype=np.uint8)
    data = b"P6 # c1\n4\n# c2\n3 255\n" + bytes(px)
    want = px.reshape(3, 4, 3).transpose(2, 0, 1).astype(np.float32) / np.float32(255.0)
    assert np.array_equal(reference_decode(data).view(np.uint32), want.view(np.uint32))


# ------------------------------------------------------------------ device paths

def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


@pytest.mark.gpu
def test_ppm_batch_decoded_on_device_bitwise():
    torch = _cuda()
    rng = np.random.default_rng(11)
    imgs = [ppm_bytes(33, 17, rng.integers(0, 256, size=33 * 17 * 3, dtype=np.uint8)) for _ in range(3)]
    d = T.load_ppm_batch(imgs)
    want = np.stack([reference_decode(b) for b in imgs])
    assert d.shape == (3, 3, 17, 33) and d.dtype == torch.float32
    assert np.array_equal(d.cpu().numpy().view(np.uint32), want.view(np.uint32))
    b16 = T.load_ppm_batch(imgs[1:2], dtype=torch.bfloat16)
    assert torch.equal(b16[0].cpu(), torch.from_numpy(want[1]).to(torch.bfloat16))
    with pytest.raises(T.FormatError):
        T.load_ppm_batch([imgs[0], ppm_bytes(2, 2, [0] * 12)])


@pytest.mark.gpu
@pytest.mark.parametrize("h,w,n,pad,c_out", [(24, 40, 5, 2, 1), (224, 224, 3, 2, 1), (31, 17, 4, 1, 3), (9, 13, 7, 3, 2)])
def test_fused_image_layer_bitwise(tmp_path, h, w, n, pad, c_out):
    """paper 4.1 path: PPM files -> u8 payload on the device -> one segregated layer with the decode
    in the kernel's loads; bitwise the same layer on the decoded batch, and the oracle's gate"""
    torch = _cuda()
    import paper_2502_20493_b200 as P
    rng = np.random.default_rng(h * w + n)
    paths = []
    for i in range(3):
        p = tmp_path / f"img{i}.ppm"
        p.write_bytes(ppm_bytes(w, h, rng.integers(0, 256, size=w * h * 3, dtype=np.uint8)))
        paths.append(p)
    bank = O.gen_kernel_bank(3, c_out, n, 9)
    layer = P.prepare_layer(bank, pad)
    fused = T.forward_ppm(layer, paths)
    decoded = T.load_ppm_batch(paths)
    assert torch.equal(fused, layer.forward(decoded))
    host = np.stack([reference_decode(p.read_bytes()) for p in paths]).astype(np.float64)
    ref = O.forward_segregated_batch(host, bank.astype(np.float64), pad)
    assert O.compare(fused.cpu().numpy(), ref, 1e-5, 1e-6)["passed"]


@pytest.mark.gpu
def test_sct_to_device(tmp_path):
    torch = _cuda()
    t = O.gen_synthetic(3, 7, 5, 4)
    blob = b"SCT1" + struct.pack("<III", 3, 7, 5) + t.astype("<f4").tobytes()
    d = T.sct_to_device(blob)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), t.view(np.uint32))
    with pytest.raises(T.FormatError):
        T.sct_to_device(b"SCT1" + struct.pack("<III", 1, 2, 2) + bytes(12))
