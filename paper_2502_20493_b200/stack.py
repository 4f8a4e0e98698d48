"""Device-resident layer stacks.

The reference's GAN_SUITE (/root/reference/pkg/src/segconv/bench.py:124-139) lists the
DCGAN / GP-GAN / EB-GAN generator layers; a reference user runs such a generator as one
`layer_forward` per layer (engines.py:163-172), every intermediate a fresh host array.
`PreparedStack` chains prepared layers on the device through the C ABI's
`segb_stack_forward`: layer i's output feeds layer i+1 from a device workspace (bf16 when
the layers compute in bf16), nothing crosses PCIe between layers, and a repeated host-batch
call with the same shape replays one captured CUDA graph of the whole chain.

Per layer the arithmetic is exactly `PreparedLayer.forward`'s (same kernels, same
accumulation order), so a stack equals the layer-by-layer chain whose intermediates are
rounded to the stack's intermediate dtype (tests/test_gpu_stack.py).
"""

from __future__ import annotations

import ctypes

from . import _device, _lib
from .engines import _PIPELINE_CHUNKS, COMPUTE_DTYPES, PreparedLayer, _copy_streams, _is_torch
from .errors import ShapeError


# a host batch is chunked when its output copy is large next to the chain's compute (EB-GAN: 4.3 GB
# out; the DCGAN stack's 13 MB output chunked ran 87 -> 73 TMAC/s end to end)
_STACK_PIPELINE_MIN_BYTES = 256 << 20


class PreparedStack:
    """A chain of PreparedLayer objects (c_out of layer i == c_in of layer i+1), all prepared
    on one device. `inter_dtype`: "bf16" or "fp32" for the intermediates (default bf16 when
    every layer computes in bf16, else fp32)."""

    def __init__(self, layers, inter_dtype: str | None = None, graph: bool = True):
        layers = list(layers)
        if not layers:
            raise ValueError("a stack needs at least one layer")
        for i, L in enumerate(layers):
            if not isinstance(L, PreparedLayer):
                raise TypeError(f"stack layer {i} is not a PreparedLayer")
            if i and layers[i - 1].c_out != L.c_in:
                raise ShapeError(f"stack layer {i} expects {L.c_in} input channels, "
                                 f"layer {i - 1} produces {layers[i - 1].c_out}")
            if L.device != layers[0].device:
                raise ValueError(f"stack layer {i} is on {L.device}, layer 0 on {layers[0].device}")
        if inter_dtype is None:
            inter_dtype = "bf16" if all(L.compute == "bf16" for L in layers) else "fp32"
        if inter_dtype not in ("bf16", "fp32", "fp64"):
            raise ValueError(f"unknown intermediate dtype {inter_dtype!r}")
        self.layers = layers
        self.inter_dtype = inter_dtype
        self.device = layers[0].device
        self.c_in, self.c_out = layers[0].c_in, layers[-1].c_out
        self.graph = graph
        self._handles = (ctypes.c_void_p * len(layers))(*[L._handle.value for L in layers])
        self._ws = {}       # (batch, h, w) -> device workspace tensor
        self._graphs = {}   # (key) -> (CUDAGraph, static x, static y)

    def output_shape(self, in_h: int, in_w: int) -> tuple[int, int]:
        for L in self.layers:
            in_h, in_w = L.output_shape(in_h, in_w)
        return in_h, in_w

    def workspace_bytes(self, batch: int, in_h: int, in_w: int, x_dtype=None, y_dtype=None) -> int:
        """Device workspace of one chained forward: the ping-pong intermediates plus the largest
        per-layer forward scratch (segb_stack_workspace_bytes2)."""
        inter = COMPUTE_DTYPES[self.inter_dtype]
        xd = inter if x_dtype is None else _device.dtype_id(x_dtype)
        yd = inter if y_dtype is None else _device.dtype_id(y_dtype)
        v = ctypes.c_int64()
        _lib.check(_lib.lib().segb_stack_workspace_bytes2(
            self._handles, len(self.layers), int(batch), int(in_h), int(in_w), xd, yd, inter, ctypes.byref(v)))
        return int(v.value)

    def _workspace(self, batch, h, w, x_dtype, y_dtype):
        key = (batch, h, w, x_dtype, y_dtype)
        if key not in self._ws:
            t = _device.torch()
            nbytes = self.workspace_bytes(batch, h, w, x_dtype, y_dtype)
            self._ws[key] = t.empty(max(1, nbytes), dtype=t.uint8, device=self.device)
        return self._ws[key]

    def _chunk_graph(self, n, h, w, x_dtype, out_dtype, slot):
        """The chain over an n-sample chunk as a captured graph on static buffers (one per slot)."""
        t = _device.torch()
        key = ("chunk", n, h, w, x_dtype, out_dtype, slot)
        if key not in self._graphs:
            oh, ow = self.output_shape(h, w)
            sx = t.zeros((n, self.c_in, h, w), dtype=x_dtype, device=self.device)
            sy = t.empty((n, self.c_out, oh, ow), dtype=out_dtype, device=self.device)
            self._launch(sx, sy)  # warm-up outside the capture
            t.cuda.current_stream(self.device).synchronize()
            g = t.cuda.CUDAGraph()
            with t.cuda.graph(g):
                self._launch(sx, sy)
            self._graphs[key] = (g, sx, sy)
        return self._graphs[key]

    def _pipeline_chunk(self, b, h, w, x_dtype, out_dtype):
        """A chunk size for the host pipeline: a divisor of the batch (b / 8, / 4 or / 2) whose
        every layer dispatches exactly as the whole batch does (same kernel and tile configuration,
        hence the same bits per sample), else 0 (no chunking)."""
        t = _device.torch()
        inter = {"bf16": t.bfloat16, "fp32": t.float32, "fp64": t.float64}[self.inter_dtype]
        for nch in (_PIPELINE_CHUNKS, 4, 2):
            if b % nch or b // nch < 2:
                continue
            cs = b // nch
            ok, hi, wi = True, h, w
            for i, L in enumerate(self.layers):
                xd = x_dtype if i == 0 else inter
                yd = out_dtype if i == len(self.layers) - 1 else inter
                if L.describe_path(cs, hi, wi, xd, yd) != L.describe_path(b, hi, wi, xd, yd):
                    ok = False
                    break
                hi, wi = L.output_shape(hi, wi)
            if ok:
                return cs
        return 0

    def _forward_host_pipelined(self, xh, out_h, out_dtype, h, w, cs):
        """Host batch in, host batch out, over batch chunks of cs samples: chunk k's chain (one
        graph replay, its input copied in first) runs while chunk k-1's output is copied out on the
        copy stream (two output buffers in rotation). Every chunk dispatches as the whole batch
        (_pipeline_chunk), so the result is the whole-batch chain's, bitwise."""
        t = _device.torch()
        main = t.cuda.current_stream(self.device)
        d2h = _copy_streams(self.device)[1]
        b = int(xh.shape[0])
        out_free = [None, None]
        last = None
        start = t.cuda.Event()
        start.record(main)
        d2h.wait_event(start)
        for k, a in enumerate(range(0, b, cs)):
            e = min(b, a + cs)
            slot = k % 2
            g, sx, sy = self._chunk_graph(e - a, h, w, xh.dtype, out_dtype, slot)
            if out_free[slot] is not None:
                main.wait_event(out_free[slot])  # the copy-out of this buffer's previous chunk
            sx.copy_(xh[a:e], non_blocking=True)
            g.replay()
            done = t.cuda.Event()
            done.record(main)
            with t.cuda.stream(d2h):
                d2h.wait_event(done)
                out_h[a:e].copy_(sy, non_blocking=True)
                last = t.cuda.Event()
                last.record(d2h)
            out_free[slot] = last
        main.wait_event(last)

    def _launch(self, d_x, d_y):
        b, _, h, w = d_x.shape
        ws = self._workspace(int(b), int(h), int(w), d_x.dtype, d_y.dtype)
        _lib.check(_lib.lib().segb_stack_forward(
            self._handles, len(self.layers), d_x.data_ptr(), _device.dtype_id(d_x.dtype), int(b), int(h), int(w),
            d_y.data_ptr(), _device.dtype_id(d_y.dtype), COMPUTE_DTYPES[self.inter_dtype], ws.data_ptr(),
            ws.numel(), _device.stream_ptr(self.device)))

    def forward(self, x, out=None, out_dtype=None):
        """x: torch (B, c_in, H, W) on the device or on the host (pinned for async copies), or
        (c_in, H, W). Returns (B, c_out, M_h, M_w) (or writes `out=`, device or host). A host
        input is copied in once and the result copied out once."""
        t = _device.require_cuda()
        if not _is_torch(x):
            raise TypeError("PreparedStack.forward takes torch tensors")
        squeeze = x.dim() == 3
        xb = x[None] if squeeze else x
        if xb.dim() != 4 or xb.shape[1] != self.c_in:
            raise ShapeError(f"stack input must be (B, {self.c_in}, H, W), got {tuple(x.shape)}")
        b, _, h, w = (int(v) for v in xb.shape)
        oh, ow = self.output_shape(h, w)
        first = self.layers[0]
        if out_dtype is None:
            out_dtype = out.dtype if out is not None else (
                t.bfloat16 if first.compute == "bf16" and xb.dtype == t.bfloat16 else
                (t.float64 if self.layers[-1].compute == "fp64" else t.float32))
        shape = (b, self.c_out, oh, ow)
        if out is not None and (tuple(out.shape) not in (shape, shape[1:] if squeeze else shape)
                                or not out.is_contiguous() or out.dtype != out_dtype):
            raise ShapeError(f"out must be a contiguous {shape} {out_dtype} tensor, got "
                             f"{tuple(out.shape)} {out.dtype}")
        host_in = not xb.is_cuda
        host_out = out is not None and not out.is_cuda
        cs = (self._pipeline_chunk(b, h, w, xb.dtype, out_dtype) if (
            host_in and host_out and self.graph and b * self.c_out * oh * ow * out.element_size() >= _STACK_PIPELINE_MIN_BYTES)
              else 0)
        if cs:
            self._forward_host_pipelined(xb, out.view(shape), out_dtype, h, w, cs)
            t.cuda.current_stream(self.device).synchronize()
            return out
        if host_in and self.graph:
            # host batch: one H2D into a static device input, the chain replayed as one
            # captured graph, one D2H of the final output
            key = (b, h, w, xb.dtype, out_dtype)
            if key not in self._graphs:
                sx = t.empty(tuple(xb.shape), dtype=xb.dtype, device=self.device)
                sy = t.empty(shape, dtype=out_dtype, device=self.device)
                sx.copy_(xb)
                self._launch(sx, sy)  # warm-up outside the capture
                t.cuda.current_stream(self.device).synchronize()
                g = t.cuda.CUDAGraph()
                with t.cuda.graph(g):
                    self._launch(sx, sy)
                self._graphs[key] = (g, sx, sy)
            g, sx, sy = self._graphs[key]
            sx.copy_(xb, non_blocking=True)
            g.replay()
            d_y = sy
        else:
            if host_in:
                xb = xb.to(self.device, non_blocking=True)
            elif xb.device != self.device:
                raise ValueError(f"input on {xb.device}, stack prepared on {self.device}")
            d_y = out.view(shape) if (out is not None and not host_out) else t.empty(
                shape, dtype=out_dtype, device=self.device)
            self._launch(xb.contiguous(), d_y)
        if out is not None:
            if out.data_ptr() != d_y.data_ptr():
                out.view(shape).copy_(d_y, non_blocking=True)
            if host_out:
                t.cuda.current_stream(self.device).synchronize()
            return out
        y = d_y.to("cpu") if host_in else d_y
        return y[0] if squeeze else y


def prepare_stack(layers, inter_dtype: str | None = None, graph: bool = True) -> PreparedStack:
    return PreparedStack(layers, inter_dtype, graph)
