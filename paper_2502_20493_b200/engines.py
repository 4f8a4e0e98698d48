"""Drop-in operator API of the segregated transpose convolution, on the B200.

Mirrors /root/reference/pkg/src/segconv/engines.py -- same names, argument
meaning and error behaviour -- with the arithmetic on the GPU through the
C ABI (include/segb200.h):

  prepare_layer / PreparedLayer.__init__   engines.py:153-160, 213-244  -> segb_prepare (K1)
  PreparedLayer.forward                    engines.py:246-256, 271-291  -> segb_forward (K2 / K3)
  layer_forward                            engines.py:163-172
  transpose_conv_segregated                engines.py:143-150
  transpose_conv_reference (Alg. 1)        engines.py:134-140 (the GPU reference engine)
  compare_outputs / ComparisonReport       engines.py:99-118, 175-198 (host-side verdict)
  EngineCounters, transpose_conv_{reference,segregated}_counted
                                           engines.py:121-126, 353-406 -> segb_counted_forward

Extensions over the reference (documented in DESIGN.md): forward also takes
torch tensors, CUDA-resident (C,H,W) or batched (B,C,H,W), returning a torch
tensor on the same device (or writing into `out=`); a CPU torch tensor (e.g.
pinned) is copied in and the result copied back; `compute="bf16"` selects
bf16 operands with fp32 accumulation (tensor cores where eligible).
There is no CPU fallback: without the CUDA library or a GPU these raise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .errors import ShapeError, SpecError
from .segregation import SubKernelSet, merge_subkernels, require_square_kernel
from .spec import TransposeConvSpec, output_dims, _spec_dims

ENGINE_REFERENCE = "reference"
ENGINE_SEGREGATED = "segregated"
ENGINES = (ENGINE_REFERENCE, ENGINE_SEGREGATED)

COMPUTE_DTYPES = {"fp32": _lib.F32, "fp64": _lib.F64, "bf16": _lib.BF16}

# host-resident batches at least this large are copied in, computed and copied out as an
# overlapped pipeline of _PIPELINE_CHUNKS batch chunks (PreparedLayer._forward_host_pipelined)
_PIPELINE_MIN_BYTES = 8 << 20
_PIPELINE_CHUNKS = 8
_COPY_STREAMS: dict = {}


def _copy_streams(dev):
    """Per-device H2D and D2H copy streams of the host pipeline (created once)."""
    key = str(dev)
    if key not in _COPY_STREAMS:
        t = _device.torch()
        _COPY_STREAMS[key] = (t.cuda.Stream(dev), t.cuda.Stream(dev))
    return _COPY_STREAMS[key]


def wait_host_copies(device=None):
    """Orders the current stream of `device` after every host copy that forwards with
    `non_blocking=True` left in flight (the pipelined host path's copy streams); after it, an event
    recorded on the current stream marks those copies complete."""
    t = _device.torch()
    dev = t.device("cuda", t.cuda.current_device()) if device is None else t.device(device)
    key = str(dev)
    if key in _COPY_STREAMS:
        cur = t.cuda.current_stream(dev)
        for s in _COPY_STREAMS[key]:
            cur.wait_stream(s)


@dataclass(frozen=True)
class ComparisonReport:
    """Element-wise agreement between two tensors (the second one is the reference)."""

    shapes_match: bool
    max_abs_diff: float | None
    max_rel_diff: float | None
    rel_tol: float
    abs_tol: float
    passed: bool

    def to_dict(self) -> dict:
        return {"shapes_match": self.shapes_match, "max_abs_diff": self.max_abs_diff,
                "max_rel_diff": self.max_rel_diff, "rel_tol": self.rel_tol,
                "abs_tol": self.abs_tol, "passed": self.passed}


def compare_outputs(a, b, rel_tol: float = 1e-5, abs_tol: float = 1e-6) -> ComparisonReport:
    """engines.py:175-198: pass iff |a - b| <= abs_tol + rel_tol * |b| everywhere."""
    a = _as_numpy(a)
    b = _as_numpy(b)
    if a.shape != b.shape:
        return ComparisonReport(False, None, None, rel_tol, abs_tol, False)
    a64 = a.astype(np.float64, copy=False)
    b64 = b.astype(np.float64, copy=False)
    d = np.abs(a64 - b64)
    den = np.maximum(np.abs(a64), np.abs(b64))
    rel = np.divide(d, den, out=np.zeros_like(d), where=den > 0)
    passed = bool(np.all(d <= abs_tol + rel_tol * np.abs(b64)))
    return ComparisonReport(True, float(d.max()) if d.size else 0.0,
                            float(rel.max()) if rel.size else 0.0, rel_tol, abs_tol, passed)


def _as_numpy(a):
    if isinstance(a, np.ndarray):
        return a
    mod = type(a).__module__
    if mod.startswith("torch"):
        return a.detach().float().cpu().numpy() if a.dtype == _device.torch().bfloat16 \
            else a.detach().cpu().numpy()
    return np.asarray(a)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def require_channel_tensor(arr, what: str = "channel tensor"):
    """tensors.py:52-60 (numpy), extended to torch (C,H,W) / (B,C,H,W)."""
    if _is_torch(arr):
        t = _device.torch()
        if arr.dim() not in (3, 4):
            raise ShapeError(f"{what} must be a 3-D (channels, height, width) or 4-D batched "
                             f"tensor, got {tuple(arr.shape)}")
        if min(arr.shape) < 1:
            raise ShapeError(f"{what} dimensions must all be >= 1, got {tuple(arr.shape)}")
        if arr.dtype not in (t.float32, t.float64, t.bfloat16):
            raise ShapeError(f"{what} must hold floats, got dtype {arr.dtype}")
        return arr
    if not isinstance(arr, np.ndarray) or arr.ndim != 3:
        raise ShapeError(f"{what} must be a 3-D (channels, height, width) array, "
                         f"got {getattr(arr, 'shape', type(arr))}")
    if min(arr.shape) < 1:
        raise ShapeError(f"{what} dimensions must all be >= 1, got {arr.shape}")
    if not np.issubdtype(arr.dtype, np.floating):
        raise ShapeError(f"{what} must hold floats, got dtype {arr.dtype}")
    return arr


class PreparedLayer:
    """A kernel bank laid out on the device for one engine (engines.py:204-244).

    Construction validates like the reference, uploads the (c_in, c_out, n, n)
    bank and runs K1 (segb_prepare): the parity split into the four class
    sub-banks, in the operand layout of the kernel that will consume them.
    Immutable afterwards and safe to share across threads and streams.
    """

    def __init__(self, bank, pad: int, engine: str = ENGINE_SEGREGATED, compute: str | None = None):
        t = _device.torch()
        is_t = _is_torch(bank)
        shape = tuple(bank.shape)
        if len(shape) != 4 or shape[2] != shape[3]:
            raise ShapeError(f"kernel bank must be (c_in, c_out, n, n) with square "
                             f"kernels, got shape {shape}")
        if shape[2] < 2:
            raise ShapeError(f"kernel side must be >= 2, got {shape[2]}")
        if is_t:
            if bank.dtype not in (t.float32, t.float64, t.bfloat16):
                raise ShapeError(f"kernel bank must hold floats, got dtype {bank.dtype}")
        else:
            bank = np.asarray(bank)
            if not np.issubdtype(bank.dtype, np.floating):
                raise ShapeError(f"kernel bank must hold floats, got dtype {bank.dtype}")
        if pad < 0:
            raise SpecError(f"padding must be >= 0, got {pad}")
        if engine not in ENGINES:
            raise ValueError(f"unknown engine {engine!r}, expected one of {ENGINES}")
        self.engine = engine
        self.pad = int(pad)
        self.c_in, self.c_out, self.kernel_n = shape[0], shape[1], shape[2]
        if is_t:
            self.bank_dtype = {t.float32: np.float32, t.float64: np.float64}.get(bank.dtype, np.float32)
        else:
            self.bank_dtype = bank.dtype
        if compute is None:
            compute = "fp64" if self.bank_dtype == np.float64 else "fp32"
        if compute not in COMPUTE_DTYPES:
            raise ValueError(f"unknown compute dtype {compute!r}, expected one of {tuple(COMPUTE_DTYPES)}")
        self.compute = compute
        _device.require_cuda()
        if is_t:
            d_bank = bank.detach().contiguous()
            if not d_bank.is_cuda:
                d_bank = d_bank.to(t.cuda.current_device())
        else:
            work = bank if bank.dtype in (np.float32, np.float64) else bank.astype(np.float64)
            d_bank = _device.to_device(work)
        self.device = d_bank.device
        handle = ctypes.c_void_p()
        _lib.check(_lib.lib().segb_prepare(
            d_bank.data_ptr(), _device.dtype_id(d_bank.dtype), self.c_in, self.c_out, self.kernel_n,
            self.pad, _lib.ENGINE_IDS[engine], COMPUTE_DTYPES[compute], _device.stream_ptr(self.device),
            ctypes.byref(handle)))
        self._handle = handle
        self._lib = _lib.lib()

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.segb_release(h)
            except Exception:  # interpreter shutdown
                pass
            self._handle = None

    # ------------------------------------------------------------------
    def output_shape(self, in_h: int, in_w: int) -> tuple[int, int]:
        return _spec_dims(in_h, in_w, self.kernel_n, self.pad)

    def select_path(self, x_dtype_id: int, batch: int, in_h: int, in_w: int,
                    compute: str | None = None) -> str:
        cid = COMPUTE_DTYPES[compute or self.compute]
        p = self._lib.segb_select_path(self._handle, x_dtype_id, batch, in_h, in_w, cid)
        return {1: "direct", 2: "igemm"}[p]

    def forward(self, x, threads: int = 1, out=None, path: str = "auto", out_dtype=None,
                non_blocking: bool = False):
        """engines.py:246-256. numpy (C,H,W) in -> numpy out (dtype = result_type of
        x and bank, as the reference); torch in -> torch out. A host `out=` tensor is complete
        when forward returns (the reference returns finished host arrays); `non_blocking=True`
        leaves that device-to-host copy in flight instead: on the caller's current stream, or -- for a
        pipelined host batch -- on the layer's copy stream, so the next call's input copies and kernels
        overlap it; `wait_host_copies()` (or a synchronize) orders the caller after it."""
        x = require_channel_tensor(x)
        c_axis = 1 if (_is_torch(x) and x.dim() == 4) else 0
        if x.shape[c_axis] != self.c_in:
            raise ShapeError(f"channel mismatch: input has {x.shape[c_axis]} channels, "
                             f"bank expects {self.c_in}")
        if threads < 1:
            raise ValueError(f"threads must be >= 1, got {threads}")
        in_h, in_w = int(x.shape[-2]), int(x.shape[-1])
        out_h, out_w = self.output_shape(in_h, in_w)
        if path not in _lib.PATH_IDS:
            raise ValueError(f"unknown path {path!r}, expected one of {tuple(_lib.PATH_IDS)}")
        if _is_torch(x):
            y = self._forward_torch(x, out, path, out_dtype, out_h, out_w, in_flight=non_blocking)
            if out is not None and not out.is_cuda and not non_blocking:
                _device.torch().cuda.current_stream(self.device).synchronize()
            return y
        return self._forward_numpy(x, out_h, out_w, path)

    def _compute_for(self, x_dt) -> str:
        if self.compute == "bf16":
            return "bf16"
        t = _device.torch()
        if x_dt in (np.float64, t.float64) or self.bank_dtype == np.float64:
            return "fp64"
        return "fp32"

    def _forward_numpy(self, x: np.ndarray, out_h: int, out_w: int, path: str) -> np.ndarray:
        t = _device.torch()
        dt = np.result_type(x.dtype, self.bank_dtype)
        compute = self._compute_for(np.float64 if dt == np.float64 else np.float32)
        host_dt = np.float64 if compute == "fp64" else np.float32
        d_x = _device.to_device(x.astype(host_dt, copy=False)[None], self.device)
        d_y = t.empty((1, self.c_out, out_h, out_w), dtype=_device.torch_dtype(_device.dtype_id(host_dt)),
                      device=self.device)
        self._launch(d_x, d_y, compute, path)
        return d_y[0].cpu().numpy().astype(dt, copy=False)

    def _forward_torch(self, x, out, path, out_dtype, out_h, out_w, in_flight=False):
        t = _device.torch()
        squeeze = x.dim() == 3
        xb = x[None] if squeeze else x
        host_in = not xb.is_cuda
        if (host_in and xb.shape[0] >= 2 and (out is None or not out.is_cuda)
                and xb.numel() * xb.element_size() >= _PIPELINE_MIN_BYTES):
            y = self._forward_host_pipelined(xb, None if out is None else out.view(
                (xb.shape[0], self.c_out, out_h, out_w)), path, out_dtype, out_h, out_w,
                in_flight=in_flight and out is not None)
            if out is not None:
                return out
            return y[0] if squeeze else y
        if host_in:
            xb = xb.to(self.device, non_blocking=True)
        elif xb.device != self.device:
            raise ValueError(f"input on {xb.device}, layer prepared on {self.device}")
        xb = xb.contiguous()
        compute = self._compute_for(xb.dtype)
        if compute == "fp64" and xb.dtype != t.float64:
            xb = xb.double()
        if compute == "fp32" and xb.dtype != t.float32:
            xb = xb.float()
        if out_dtype is None:
            out_dtype = (out.dtype if out is not None else
                         (t.bfloat16 if compute == "bf16" and xb.dtype == t.bfloat16 else
                          (t.float64 if compute == "fp64" else t.float32)))
        shape = (xb.shape[0], self.c_out, out_h, out_w)
        if out is not None and out.is_cuda:
            if tuple(out.shape) not in (shape, shape[1:] if squeeze else shape) or not out.is_contiguous():
                raise ShapeError(f"out must be a contiguous {shape} tensor, got {tuple(out.shape)}")
            if out.dtype != out_dtype:
                raise ValueError(f"out dtype {out.dtype} != {out_dtype}")
            d_y = out.view(shape)
        else:
            d_y = t.empty(shape, dtype=out_dtype, device=self.device)
        self._launch(xb, d_y, compute, path)
        if out is not None and not out.is_cuda:
            out.view(shape).copy_(d_y, non_blocking=True)
            return out
        if host_in:
            return (d_y[0] if squeeze else d_y).to("cpu")
        return d_y[0] if squeeze else d_y

    def _pipeline_chunk(self, b, h, w, x_dtype, y_dtype, compute, path):
        """Chunk size of the host pipeline: b / 8, / 4 or / 2 (rounded up), the first whose chunk
        sizes all dispatch exactly as the whole batch (same kernel and tile configuration, so the
        same bits per sample: the dispatch adapts to the batch, e.g. split K for small ones), else
        the whole batch as one chunk."""
        whole = self.describe_path(b, h, w, x_dtype, y_dtype, compute, path)
        for nch in (_PIPELINE_CHUNKS, 4, 2):
            cs = (b + nch - 1) // nch
            if cs < 1 or cs >= b:
                continue
            sizes = {cs, b - cs * ((b - 1) // cs)}
            if all(self.describe_path(n, h, w, x_dtype, y_dtype, compute, path) == whole for n in sizes):
                return cs
        return b

    def _forward_host_pipelined(self, xh, out_h_t, path, out_dtype, out_h, out_w, in_flight=False):
        """Host (pinned) batch in, host batch out, as a 3-stage pipeline over batch chunks:
        the H2D copy of chunk k+1 (copy stream), the kernels of chunk k (caller's stream) and
        the D2H copy of chunk k-1 (second copy stream) overlap, so PCIe runs both directions at
        once instead of copy-in / compute / copy-out in series. The chunks dispatch as the whole
        batch does (_pipeline_chunk), so the result is bitwise that of one whole-batch call. Ordered after prior work on the
        caller's current stream, which waits for the last copy before returning; a returned
        (not `out=`) tensor is complete on return, as `.to("cpu")` would be."""
        t = _device.torch()
        dev = self.device
        main = t.cuda.current_stream(dev)
        h2d, d2h = _copy_streams(dev)
        b = int(xh.shape[0])
        compute = self._compute_for(xh.dtype)
        dev_in_dt = {"fp64": t.float64, "fp32": t.float32}.get(compute, xh.dtype)
        if out_dtype is None:
            out_dtype = (out_h_t.dtype if out_h_t is not None else
                         (t.bfloat16 if compute == "bf16" and xh.dtype == t.bfloat16 else
                          (t.float64 if compute == "fp64" else t.float32)))
        shape = (b, self.c_out, out_h, out_w)
        returned = out_h_t is None
        if returned:
            out_h_t = t.empty(shape, dtype=out_dtype, pin_memory=True)
        elif tuple(out_h_t.shape) != shape or not out_h_t.is_contiguous():
            raise ShapeError(f"out must be a contiguous {shape} tensor, got {tuple(out_h_t.shape)}")
        elif out_h_t.dtype != out_dtype:
            raise ValueError(f"out dtype {out_h_t.dtype} != {out_dtype}")
        cs = self._pipeline_chunk(b, xh.shape[-2], xh.shape[-1], dev_in_dt, out_dtype, compute, path)
        spans = [(i, min(b, i + cs)) for i in range(0, b, cs)]
        xin = [t.empty((cs,) + tuple(xh.shape[1:]), dtype=xh.dtype, device=dev) for _ in range(2)]
        yout = [t.empty((cs,) + shape[1:], dtype=out_dtype, device=dev) for _ in range(2)]
        start = t.cuda.Event()
        start.record(main)
        h2d.wait_event(start)
        d2h.wait_event(start)
        in_free = [None, None]
        out_free = [None, None]
        last = None
        for k, (a, e) in enumerate(spans):
            slot, n = k % 2, e - a
            with t.cuda.stream(h2d):
                if in_free[slot] is not None:
                    h2d.wait_event(in_free[slot])
                xin[slot][:n].copy_(xh[a:e], non_blocking=True)
                in_ready = t.cuda.Event()
                in_ready.record(h2d)
            main.wait_event(in_ready)
            if out_free[slot] is not None:
                main.wait_event(out_free[slot])
            xd = xin[slot][:n]
            if xd.dtype != dev_in_dt:
                xd = xd.to(dev_in_dt)
            self._launch(xd, yout[slot][:n], compute, path)
            done = t.cuda.Event()
            done.record(main)
            in_free[slot] = done
            with t.cuda.stream(d2h):
                d2h.wait_event(done)
                out_h_t[a:e].copy_(yout[slot][:n], non_blocking=True)
                last = t.cuda.Event()
                last.record(d2h)
                out_free[slot] = last
        for buf in xin:
            buf.record_stream(h2d)
        for buf in yout:
            buf.record_stream(d2h)
        if not in_flight:  # (in flight: wait_host_copies() orders the caller after the copies)
            main.wait_event(last)
        main.wait_event(in_ready)
        if returned:
            main.synchronize()
        return out_h_t

    def describe_path(self, batch: int, in_h: int, in_w: int, x_dtype=None, y_dtype=None,
                      compute: str | None = None, path: str = "auto") -> str:
        """The kernel family (and operand mode) a forward of this shape runs (segb_describe_path)."""
        t = _device.torch()
        compute = compute or self.compute
        if x_dtype is None:
            x_dtype = t.bfloat16 if compute == "bf16" else (t.float64 if compute == "fp64" else t.float32)
        if y_dtype is None:
            y_dtype = x_dtype
        buf = ctypes.create_string_buffer(128)
        _lib.check(self._lib.segb_describe_path(self._handle, _device.dtype_id(x_dtype), int(batch), int(in_h),
                                                int(in_w), _device.dtype_id(y_dtype), COMPUTE_DTYPES[compute],
                                                _lib.PATH_IDS[path], buf, 128))
        return buf.value.decode()

    def workspace_bytes(self, batch: int, in_h: int, in_w: int, x_dtype=None, y_dtype=None,
                        compute: str | None = None, path: str = "auto") -> int:
        """Device scratch bytes one forward of this shape takes (segb_forward_workspace_bytes):
        K3's channels-last operand copy or K3c's tap products; 0 for K2 and K3b."""
        t = _device.torch()
        compute = compute or self.compute
        if x_dtype is None:
            x_dtype = t.bfloat16 if compute == "bf16" else (t.float64 if compute == "fp64" else t.float32)
        if y_dtype is None:
            y_dtype = x_dtype
        return self._ws_bytes(_device.dtype_id(x_dtype), _device.dtype_id(y_dtype), int(batch), int(in_h),
                              int(in_w), COMPUTE_DTYPES[compute], _lib.PATH_IDS[path])

    def _ws_bytes(self, xd, yd, b, h, w, cid, pid) -> int:
        # not cached: the kernel choice (and so the scratch) can follow A/B environment switches
        r = ctypes.c_int64()
        _lib.check(self._lib.segb_forward_workspace_bytes(self._handle, xd, b, h, w, yd, cid, pid, ctypes.byref(r)))
        return int(r.value)

    def _launch(self, d_x, d_y, compute: str, path: str) -> None:
        """One segb_forward_ws call on the caller's current stream. The workspace (if the kernel
        needs one) comes from torch's stream-ordered caching allocator on the layer's device, so
        the C ABI never allocates and concurrent streams never share scratch."""
        b, _, h, w = d_x.shape
        xd, yd = _device.dtype_id(d_x.dtype), _device.dtype_id(d_y.dtype)
        cid, pid = COMPUTE_DTYPES[compute], _lib.PATH_IDS[path]
        nbytes = self._ws_bytes(xd, yd, int(b), int(h), int(w), cid, pid)
        ws = _device.torch().empty(nbytes, dtype=_device.torch().uint8, device=self.device) if nbytes else None
        _lib.check(self._lib.segb_forward_ws(
            self._handle, d_x.data_ptr(), xd, int(b), int(h), int(w), d_y.data_ptr(), yd, cid, pid,
            ws.data_ptr() if ws is not None else None, nbytes, _device.stream_ptr(self.device)))


def prepare_layer(bank, pad: int, engine: str = ENGINE_SEGREGATED, compute: str | None = None) -> PreparedLayer:
    """engines.py:153-160: lay out a (c_in, c_out, n, n) bank once for repeated forwards."""
    return PreparedLayer(bank, pad, engine, compute)


def layer_forward(x, bank, pad: int, engine: str = ENGINE_SEGREGATED, threads: int = 1,
                  compute: str | None = None):
    """engines.py:163-172: out[co] = sum_ci tconv(x[ci], bank[ci, co], pad)."""
    return prepare_layer(bank, pad, engine, compute).forward(x, threads=threads)


def require_feature_map(arr, what: str = "feature map") -> np.ndarray:
    """tensors.py:42-49."""
    if not isinstance(arr, np.ndarray) or arr.ndim != 2:
        raise ShapeError(f"{what} must be a 2-D array, got {getattr(arr, 'shape', type(arr))}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ShapeError(f"{what} must be at least 1x1, got {arr.shape}")
    if not np.issubdtype(arr.dtype, np.floating):
        raise ShapeError(f"{what} must hold floats, got dtype {arr.dtype}")
    return arr


def transpose_conv_segregated(feature_map, subs: SubKernelSet, pad: int) -> np.ndarray:
    """engines.py:143-150: single map through merge -> prepare -> forward."""
    m = require_feature_map(feature_map)
    _spec_dims(m.shape[0], m.shape[1], subs.size, pad)
    bank = merge_subkernels(subs)[np.newaxis, np.newaxis]
    return prepare_layer(bank, pad, ENGINE_SEGREGATED).forward(m[np.newaxis])[0]


def transpose_conv_reference(feature_map, kernel, pad: int) -> np.ndarray:
    """engines.py:134-140: Alg. 1 (upsample -> pad P -> correlate), evaluated on the GPU."""
    m = require_feature_map(feature_map)
    k = require_square_kernel(kernel)
    _spec_dims(m.shape[0], m.shape[1], k.shape[0], pad)
    return prepare_layer(k[np.newaxis, np.newaxis], pad, ENGINE_REFERENCE).forward(m[np.newaxis])[0]


@dataclass
class EngineCounters:
    """engines.py:121-126: operation counts recorded by the instrumented scalar engines."""

    mults: int = 0
    writes: int = 0


def _counted(m: np.ndarray, k: np.ndarray, pad: int, engine: str):
    """segb_counted_forward on one map: fp64 output and the kernel's own mults/writes counts."""
    t = _device.require_cuda()
    h, w = m.shape
    oh, ow = _spec_dims(h, w, k.shape[0], pad)
    mw = m if m.dtype in (np.float32, np.float64) else m.astype(np.float64)
    kw = k if k.dtype in (np.float32, np.float64) else k.astype(np.float64)
    dev = t.cuda.current_device()
    d_m = _device.to_device(mw, dev)
    d_k = _device.to_device(kw, dev)
    d_out = t.empty((oh, ow), dtype=t.float64, device=dev)
    d_cnt = t.zeros(2, dtype=t.int64, device=dev)
    _lib.check(_lib.lib().segb_counted_forward(
        d_m.data_ptr(), _device.dtype_id(d_m.dtype), int(h), int(w), d_k.data_ptr(), _device.dtype_id(d_k.dtype),
        int(k.shape[0]), int(pad), _lib.ENGINE_IDS[engine], d_out.data_ptr(), d_cnt.data_ptr(),
        _device.stream_ptr(dev)))
    cnt = d_cnt.cpu().tolist()
    return d_out.cpu().numpy(), EngineCounters(mults=int(cnt[0]), writes=int(cnt[1]))


def transpose_conv_reference_counted(feature_map, kernel, pad: int):
    """engines.py:353-376: Alg. 1 per element (upsample, pad P, all n x n taps) with counters."""
    m = require_feature_map(feature_map)
    k = require_square_kernel(kernel)
    _spec_dims(m.shape[0], m.shape[1], k.shape[0], pad)
    return _counted(m, k, pad, ENGINE_REFERENCE)


def transpose_conv_segregated_counted(feature_map, subs: SubKernelSet, pad: int):
    """engines.py:379-406: the unified rule per element (one parity sub-kernel per output) with
    counters. The sub-kernels are merged back into K (bit-exact, segregation.py:73-88); the
    device kernel reads k_rs[u, v] as K[2u + r, 2v + s]."""
    m = require_feature_map(feature_map)
    _spec_dims(m.shape[0], m.shape[1], subs.size, pad)
    return _counted(m, merge_subkernels(subs), pad, ENGINE_SEGREGATED)


__all__ = [
    "ENGINE_REFERENCE", "ENGINE_SEGREGATED", "ENGINES", "ComparisonReport", "EngineCounters", "PreparedLayer",
    "SpecError", "ShapeError", "TransposeConvSpec", "compare_outputs", "layer_forward",
    "output_dims", "prepare_layer", "transpose_conv_reference", "transpose_conv_reference_counted",
    "transpose_conv_segregated", "transpose_conv_segregated_counted",
]
