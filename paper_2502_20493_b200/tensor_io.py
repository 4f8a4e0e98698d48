"""Dataset inputs to the device: binary PPM (P6) images and SCT1 tensors.

Mirrors /root/reference/pkg/src/segconv/tensor_io.py -- same names, header rules, messages and
`FormatError` -- for the host-side decode, and adds device loaders for the paper's dataset path
(§4.1: 224x224x3 images through a single-map layer):

  parse_ppm / load_ppm                 tensor_io.py:27-58 (host, numpy, bitwise the reference)
  tensor_to_sct_bytes / sct_bytes_to_tensor / save_raw_tensor / load_raw_tensor   :61-100
  ppm_to_device / load_ppm_batch       header parsed on the host, only the raw u8 payload copied
                                       up, deinterleaved + scaled by segb_u8_hwc_to_chw (bitwise
                                       the host decode)
  sct_to_device                        SCT1 payload (already f32 CHW) copied up as is

The device loaders return torch tensors ready for `PreparedLayer.forward` (a batch of images is
one (B, 3, H, W) tensor).
"""

from __future__ import annotations

import struct

import numpy as np

from . import _device, _lib
from .engines import require_channel_tensor

SCT_MAGIC = b"SCT1"
_PPM_WHITESPACE = b" \t\r\n\x0b\x0c"


class FormatError(ValueError):
    """A file's bytes do not match the declared format (tensor_io.py:24-25)."""


def _ppm_token(data: bytes, pos: int) -> tuple[bytes, int]:
    # tensor_io.py:103-118: skip whitespace and '#' comments, then collect one token
    while pos < len(data):
        byte = data[pos]
        if byte in _PPM_WHITESPACE:
            pos += 1
        elif byte == ord("#"):
            while pos < len(data) and data[pos] not in b"\r\n":
                pos += 1
        else:
            break
    if pos >= len(data):
        raise FormatError("malformed PPM header: unexpected end of data")
    start = pos
    while pos < len(data) and data[pos] not in _PPM_WHITESPACE:
        pos += 1
    return data[start:pos], pos


def _ppm_payload(data: bytes) -> tuple[memoryview, int, int]:
    """tensor_io.py:27-51 header rules -> (u8 payload of height*width*3 bytes, height, width)."""
    magic, pos = _ppm_token(data, 0)
    if magic != b"P6":
        raise FormatError(f"unsupported PPM magic {magic!r}, only binary P6 is handled")
    fields = []
    for name in ("width", "height", "maxval"):
        token, pos = _ppm_token(data, pos)
        try:
            fields.append(int(token))
        except ValueError:
            raise FormatError(f"malformed PPM header: non-numeric {name} {token!r}") from None
    width, height, maxval = fields
    if width < 1 or height < 1:
        raise FormatError(f"malformed PPM header: size {width}x{height}")
    if maxval != 255:
        raise FormatError(f"unsupported PPM maxval {maxval}, expected 255")
    if pos >= len(data) or data[pos] not in _PPM_WHITESPACE:
        raise FormatError("malformed PPM header: missing whitespace before pixel data")
    pos += 1
    expected = width * height * 3
    payload = memoryview(data)[pos:pos + expected]
    if len(payload) < expected:
        raise FormatError(f"truncated PPM pixel data: expected {expected} bytes, got {len(payload)}")
    return payload, height, width


def parse_ppm(data: bytes) -> np.ndarray:
    """Decode binary P6 bytes into a (3, height, width) float32 tensor in [0, 1] (host)."""
    payload, height, width = _ppm_payload(data)
    pixels = np.frombuffer(payload, dtype=np.uint8).reshape(height, width, 3)
    return pixels.transpose(2, 0, 1).astype(np.float32) / np.float32(255.0)


def load_ppm(path) -> np.ndarray:
    with open(path, "rb") as fh:
        return parse_ppm(fh.read())


def tensor_to_sct_bytes(tensor) -> bytes:
    """Serialize a (C, H, W) channel tensor to SCT1 bytes (tensor_io.py:61-66)."""
    t = require_channel_tensor(np.asarray(tensor))
    channels, height, width = t.shape
    return SCT_MAGIC + struct.pack("<III", channels, height, width) + np.ascontiguousarray(t, dtype="<f4").tobytes()


def _sct_header(data: bytes) -> tuple[int, int, int]:
    if len(data) < 16:
        raise FormatError(f"SCT1 data too short for header: {len(data)} bytes")
    if data[:4] != SCT_MAGIC:
        raise FormatError(f"bad magic {bytes(data[:4])!r}, expected {SCT_MAGIC!r}")
    channels, height, width = struct.unpack("<III", data[4:16])
    if channels < 1 or height < 1 or width < 1:
        raise FormatError(f"invalid SCT1 dims {channels}x{height}x{width}")
    expected = channels * height * width * 4
    if len(data) - 16 != expected:
        raise FormatError(f"SCT1 payload size mismatch: header implies {expected} bytes, got {len(data) - 16}")
    return channels, height, width


def sct_bytes_to_tensor(data: bytes) -> np.ndarray:
    """Parse SCT1 bytes back into a (channels, height, width) float32 tensor (tensor_io.py:69-84)."""
    c, h, w = _sct_header(data)
    return np.frombuffer(data[16:], dtype="<f4").astype(np.float32).reshape(c, h, w)


def save_raw_tensor(tensor, path) -> None:
    with open(path, "wb") as fh:
        fh.write(tensor_to_sct_bytes(tensor))


def load_raw_tensor(path) -> np.ndarray:
    with open(path, "rb") as fh:
        return sct_bytes_to_tensor(fh.read())


# ---------------------------------------------------------------------------- device loaders

def _read(src) -> bytes:
    if isinstance(src, (bytes, bytearray, memoryview)):
        return bytes(src)
    with open(src, "rb") as fh:
        return fh.read()


def load_ppm_batch(sources, device=None, dtype=None):
    """PPM files or byte strings (all the same size) -> one (B, 3, H, W) device tensor,
    bitwise `np.stack([parse_ppm(s) for s in sources])` (fp32; `dtype` bf16 / fp64 converts
    that value). Only the u8 payloads are copied to the device."""
    t = _device.require_cuda()
    dtype = dtype or t.float32
    payloads, dims = [], None
    for s in sources:
        payload, h, w = _ppm_payload(_read(s))
        if dims is not None and (h, w) != dims:
            raise FormatError(f"PPM batch mixes sizes {dims[0]}x{dims[1]} and {h}x{w}")
        dims = (h, w)
        payloads.append(np.frombuffer(payload, dtype=np.uint8))
    if dims is None:
        raise ValueError("load_ppm_batch needs at least one image")
    h, w = dims
    host = t.from_numpy(np.concatenate(payloads)).pin_memory()
    dev = device or t.device("cuda", t.cuda.current_device())
    src = host.to(dev, non_blocking=True)
    out = t.empty((len(payloads), 3, h, w), dtype=dtype, device=dev)
    _lib.check(_lib.lib().segb_u8_hwc_to_chw(src.data_ptr(), len(payloads), h, w, 3, out.data_ptr(),
                                             _device.dtype_id(dtype), _device.stream_ptr(dev)))
    return out


def ppm_to_device(src, device=None, dtype=None):
    """One PPM (path or bytes) -> (3, H, W) device tensor, bitwise `parse_ppm` (fp32)."""
    return load_ppm_batch([src], device, dtype)[0]


def sct_to_device(src, device=None):
    """One SCT1 tensor (path or bytes) -> (C, H, W) float32 device tensor."""
    t = _device.require_cuda()
    data = _read(src)
    c, h, w = _sct_header(data)
    host = t.from_numpy(np.frombuffer(data, dtype="<f4", offset=16).astype(np.float32).reshape(c, h, w))
    return host.to(device or t.device("cuda", t.cuda.current_device()))
