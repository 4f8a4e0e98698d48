"""Dataset images and tensors straight to the device (the paper's 4.1
dataset path: 224x224x3 images through a single-map layer).

The host-side formats stay the reference's (segconv.tensor_io: parse_ppm decodes a binary P6
PPM into a (3, H, W) float32 tensor, tensor_io.py:27-58; SCT1 raw tensors, :61-100). What this
module adds is the device side of that path:

  ppm_payloads(sources)            the raw interleaved u8 pixels of a batch of same-size PPMs as
                                   one (B, H, W, 3) device tensor: one H2D copy of a quarter of the
                                   fp32 bytes, nothing decoded on the host
  forward_ppm(layer, sources)      the layer on those pixels with the decode fused into the direct
                                   kernel's loads (x dtype SEGB_U8_HWC: float32(u8) / 255, IEEE
                                   division): bitwise layer.forward(stack(parse_ppm(s)))
  load_ppm_batch(sources, dtype)   the decoded (B, 3, H, W) tensor on the device (segb_u8_hwc_to_chw)
                                   for consumers other than a layer
  sct_to_device(src)               an SCT1 tensor's f32 payload copied up as is

Only the byte offset of the pixel payload is found here (a regular-expression scan of the P6
header: magic, width, height, maxval, separated by whitespace and '#' comments, one whitespace
byte before the pixels); malformed bytes raise FormatError.
"""

from __future__ import annotations

import re

import numpy as np

from . import _device, _lib

U8_HWC = 3  # segb_dtype SEGB_U8_HWC (include/segb200.h)

_SEP = rb"(?:[ \t\r\n\x0b\x0c]|#[^\r\n]*)+"
_P6 = re.compile(rb"P6" + _SEP + rb"(\S+)" + _SEP + rb"(\S+)" + _SEP + rb"(\S+)[ \t\r\n\x0b\x0c]", re.S)


class FormatError(ValueError):
    """A file's bytes do not match the declared format (the reference's tensor_io.FormatError)."""


def _bytes(src) -> bytes:
    if isinstance(src, (bytes, bytearray, memoryview)):
        return bytes(src)
    with open(src, "rb") as fh:
        return fh.read()


def ppm_geometry(data: bytes) -> tuple[int, int, int]:
    """(height, width, payload offset) of a binary P6 PPM with maxval 255."""
    if not data.startswith(b"P6"):
        raise FormatError(f"unsupported PPM magic {data[:2]!r}, only binary P6 is handled")
    m = _P6.match(data)
    if m is None:
        raise FormatError("malformed PPM header")
    try:
        width, height, maxval = (int(g) for g in m.groups())
    except ValueError:
        raise FormatError(f"malformed PPM header: non-numeric field in {m.group(0)!r}") from None
    if width < 1 or height < 1:
        raise FormatError(f"malformed PPM header: size {width}x{height}")
    if maxval != 255:
        raise FormatError(f"unsupported PPM maxval {maxval}, expected 255")
    if len(data) - m.end() < width * height * 3:
        raise FormatError(f"truncated PPM pixel data: expected {width * height * 3} bytes, "
                          f"got {len(data) - m.end()}")
    return height, width, m.end()


def ppm_payloads(sources, device=None):
    """Same-size PPMs (paths or bytes) -> (B, H, W, 3) uint8 device tensor of their pixels."""
    t = _device.require_cuda()
    blobs, dims = [], None
    for src in sources:
        data = _bytes(src)
        h, w, off = ppm_geometry(data)
        if dims is not None and (h, w) != dims:
            raise FormatError(f"PPM batch mixes sizes {dims[0]}x{dims[1]} and {h}x{w}")
        dims = (h, w)
        blobs.append(np.frombuffer(data, dtype=np.uint8, count=h * w * 3, offset=off))
    if dims is None:
        raise ValueError("a PPM batch needs at least one image")
    host = t.from_numpy(np.stack(blobs).reshape(len(blobs), dims[0], dims[1], 3)).pin_memory()
    dev = device or t.device("cuda", t.cuda.current_device())
    return host.to(dev, non_blocking=True)


def forward_ppm(layer, sources, out=None):
    """`layer` (a 3-input-channel fp32 PreparedLayer) on a batch of PPM images, the pixel decode
    fused into the direct kernel's input loads. Returns (B, c_out, M_h, M_w) fp32 on the device,
    bitwise `layer.forward` of the reference-decoded (B, 3, H, W) batch."""
    t = _device.require_cuda()
    if layer.c_in != 3:
        raise ValueError(f"PPM images have 3 channels, the layer expects {layer.c_in}")
    if layer.compute != "fp32":
        raise ValueError(f"the fused image path computes in fp32, the layer is {layer.compute}")
    px = ppm_payloads(sources, layer.device)
    b, h, w, _ = px.shape
    oh, ow = layer.output_shape(h, w)
    shape = (b, layer.c_out, oh, ow)
    if out is None:
        out = t.empty(shape, dtype=t.float32, device=layer.device)
    elif tuple(out.shape) != shape or out.dtype != t.float32 or not out.is_cuda or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {shape} float32 device tensor")
    _lib.check(layer._lib.segb_forward_ws(layer._handle, px.data_ptr(), U8_HWC, int(b), int(h), int(w),
                                          out.data_ptr(), _lib.F32, _lib.F32, _lib.PATH_IDS["direct"], None, 0,
                                          _device.stream_ptr(layer.device)))
    return out


def load_ppm_batch(sources, device=None, dtype=None):
    """PPMs -> decoded (B, 3, H, W) device tensor (fp32 by default; bf16 / fp64 convert that
    value), bitwise the reference's parse_ppm for fp32."""
    t = _device.require_cuda()
    dtype = dtype or t.float32
    px = ppm_payloads(sources, device)
    b, h, w, c = px.shape
    out = t.empty((b, c, h, w), dtype=dtype, device=px.device)
    _lib.check(_lib.lib().segb_u8_hwc_to_chw(px.data_ptr(), int(b), int(h), int(w), int(c), out.data_ptr(),
                                             _device.dtype_id(dtype), _device.stream_ptr(px.device)))
    return out


def sct_to_device(src, device=None):
    """One SCT1 tensor ("SCT1" + three little-endian u32 dims + f32 CHW payload) -> (C, H, W)
    float32 device tensor."""
    t = _device.require_cuda()
    data = _bytes(src)
    if len(data) < 16 or data[:4] != b"SCT1":
        raise FormatError("not an SCT1 tensor")
    c, h, w = (int(v) for v in np.frombuffer(data, dtype="<u4", count=3, offset=4))
    if min(c, h, w) < 1 or len(data) - 16 != c * h * w * 4:
        raise FormatError(f"SCT1 size mismatch: dims {c}x{h}x{w}, {len(data) - 16} payload bytes")
    host = t.from_numpy(np.frombuffer(data, dtype="<f4", offset=16).astype(np.float32).reshape(c, h, w))
    return host.to(device or t.device("cuda", t.cuda.current_device()))
