"""INTEGRATION.md option B, as running code: the binding a maintainer would add to the reference
package as `segconv/gpu.py`, routing its segregated engine to the B200 path through the C ABI
(include/segb200.h) -- nothing from paper_2502_20493_b200's Python layer is used, only
libsegb200.so, ctypes, and torch for device memory and the current stream.

    import segconv
    from integration import segconv_gpu
    segconv_gpu.route(segconv)      # engine "segregated" now computes on the GPU

After route(), every caller of the reference (PreparedLayer / prepare_layer / layer_forward,
transpose_conv_segregated, the harness `run_benchmark`, the service, the CLI) reaches the GPU for
the segregated engine: `PreparedLayer.__init__` (engines.py:213-244) also prepares the device
layer (segb_prepare: K1), and `PreparedLayer._forward_segregated` (engines.py:271-291) becomes one
segb_forward_ws call. The instrumented scalar engines (engines.py:353-406) are routed to
segb_counted_forward. The reference engine (Alg. 1) stays on the CPU: it is the oracle.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.environ.get("SEGB200_LIB", os.path.join(_ROOT, "paper_2502_20493_b200", "lib", "libsegb200.so"))

_F32, _F64 = 0, 1
_SEGREGATED, _REFERENCE = 1, 0
_lib = None
calls = {"prepare": 0, "forward": 0, "counted": 0}  # evidence that the GPU path ran


def _load():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB_PATH)
        p, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        L.segb_prepare.argtypes = [p, i, i, i, i, i, i, i, p, ctypes.POINTER(p)]
        L.segb_forward_workspace_bytes.argtypes = [p, i, i64, i, i, i, i, i, ctypes.POINTER(i64)]
        L.segb_forward_ws.argtypes = [p, p, i, i64, i, i, p, i, i, i, p, i64, p]
        L.segb_counted_forward.argtypes = [p, i, i, i, p, i, i, i, i, p, p, p]
        L.segb_release.argtypes = [p]
        L.segb_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc, errors):
    if rc:
        exc = {1: errors["SpecError"], 2: errors["ShapeError"], 3: ValueError}.get(rc, RuntimeError)
        raise exc(_load().segb_last_error().decode())


class GpuLayer:
    """Device side of one reference PreparedLayer(bank, pad, "segregated")."""

    def __init__(self, bank: np.ndarray, pad: int, errors):
        import torch
        self._errors = errors
        dt = _F64 if bank.dtype == np.float64 else _F32
        host = np.ascontiguousarray(bank, dtype=np.float64 if dt == _F64 else np.float32)
        self._bank = torch.from_numpy(host).cuda()
        self.c_in, self.c_out, self.n = (int(v) for v in bank.shape[:3])
        self.pad = int(pad)
        self._h = ctypes.c_void_p()
        _check(_load().segb_prepare(self._bank.data_ptr(), dt, self.c_in, self.c_out, self.n, self.pad,
                                    _SEGREGATED, dt, torch.cuda.current_stream().cuda_stream,
                                    ctypes.byref(self._h)), errors)
        calls["prepare"] += 1

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib is not None:
            _lib.segb_release(self._h)

    def forward(self, x: np.ndarray, dt) -> np.ndarray:
        """(c_in, H, W) host array -> (c_out, M_h, M_w) host array of dtype dt (the reference's
        np.result_type of x and the bank, engines.py:272); fp64 computes in fp64."""
        import torch
        code = _F64 if dt == np.float64 else _F32
        xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64 if code == _F64 else np.float32)).cuda()
        _, h, w = x.shape
        oh, ow = 2 * h + 2 * self.pad - self.n, 2 * w + 2 * self.pad - self.n
        yd = torch.empty((self.c_out, oh, ow), dtype=xd.dtype, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        need = ctypes.c_int64()
        _check(_load().segb_forward_workspace_bytes(self._h, code, 1, h, w, code, code, 0, ctypes.byref(need)),
               self._errors)
        ws = torch.empty(max(1, need.value), dtype=torch.uint8, device="cuda")
        _check(_load().segb_forward_ws(self._h, xd.data_ptr(), code, 1, h, w, yd.data_ptr(), code, code, 0,
                                       ws.data_ptr(), need.value, stream), self._errors)
        calls["forward"] += 1
        return yd.cpu().numpy().astype(dt, copy=False)


def _counted(m: np.ndarray, k: np.ndarray, pad: int, engine: int, errors, counters_cls):
    import torch
    m64 = torch.from_numpy(np.ascontiguousarray(m, dtype=np.float64)).cuda()
    k64 = torch.from_numpy(np.ascontiguousarray(k, dtype=np.float64)).cuda()
    h, w = m.shape
    n = k.shape[0]
    oh, ow = 2 * h + 2 * pad - n, 2 * w + 2 * pad - n
    out = torch.empty((max(oh, 1), max(ow, 1)), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    _check(_load().segb_counted_forward(m64.data_ptr(), _F64, h, w, k64.data_ptr(), _F64, n, pad, engine,
                                        out.data_ptr(), cnt.data_ptr(), torch.cuda.current_stream().cuda_stream),
           errors)
    calls["counted"] += 1
    c = cnt.cpu().tolist()
    return out.cpu().numpy(), counters_cls(mults=int(c[0]), writes=int(c[1]))


def route(segconv) -> None:
    """Patch the (unmodified, installed) reference so engine "segregated" runs on the GPU."""
    engines = segconv.engines
    errors = {"SpecError": engines.SpecError, "ShapeError": segconv.tensors.ShapeError}
    PL = engines.PreparedLayer
    if getattr(PL, "_segb200_routed", False):
        return
    orig_init = PL.__init__

    def __init__(self, bank, pad, engine):
        orig_init(self, bank, pad, engine)  # the reference's own validation and CPU layouts
        self._gpu = GpuLayer(np.asarray(bank), pad, errors) if engine == engines.ENGINE_SEGREGATED else None

    def _forward_segregated(self, x, out_h, out_w, threads):
        dt = np.result_type(x.dtype, self._classes[0][4].dtype)
        return self._gpu.forward(x, dt)

    PL.__init__ = __init__
    PL._forward_segregated = _forward_segregated
    PL._segb200_routed = True

    def transpose_conv_reference_counted(feature_map, kernel, pad):
        m = segconv.tensors.require_feature_map(feature_map)
        k = segconv.tensors.require_square_kernel(kernel)
        engines._check_case(m.shape[0], m.shape[1], k.shape[0], pad)
        return _counted(m, k, pad, _REFERENCE, errors, engines.EngineCounters)

    def transpose_conv_segregated_counted(feature_map, subs, pad):
        m = segconv.tensors.require_feature_map(feature_map)
        engines._check_case(m.shape[0], m.shape[1], subs.size, pad)
        k = segconv.segregation.merge_subkernels(subs)
        return _counted(m, k, pad, _SEGREGATED, errors, engines.EngineCounters)

    for mod in (engines, segconv):
        mod.transpose_conv_reference_counted = transpose_conv_reference_counted
        mod.transpose_conv_segregated_counted = transpose_conv_segregated_counted


# ------------------------------------------------------------------ GPU columns for the harness

def gpu_record(config, seed: int, index: int, batch: int = 64, compute: str = "fp32", repeats: int = 10) -> dict:
    """The "gpu" object the routed harness adds to a reference layer record:
    the layer on a device-resident batch of `batch` samples of the harness's input stream (sample 0
    is the reference's own input, bench.py:299-301), CUDA-event timed (median of `repeats`), with the
    kernel the dispatcher picked and useful GMAC/s (mult_count_segregated x batch / time)."""
    import torch

    import paper_2502_20493_b200 as P
    from paper_2502_20493_b200.synth import device_unit_floats, harness_seeds
    in_seed, bank_seed = harness_seeds(seed, index)
    dt = torch.bfloat16 if compute == "bf16" else torch.float32
    bank = device_unit_floats((config.c_in, config.c_out, config.kernel_n, config.kernel_n), bank_seed)
    layer = P.prepare_layer(bank, config.pad, compute=compute)
    x = device_unit_floats((batch, config.c_in, config.input_h, config.input_w), in_seed, dtype=dt)
    y = layer.forward(x)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(repeats)]
    for a, b in ev:
        a.record()
        layer.forward(x, out=y)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[repeats // 2]
    macs = P.mult_count_segregated(P.TransposeConvSpec(config.input_h, config.input_w, config.kernel_n,
                                                       config.pad, config.c_in, config.c_out)) * batch
    return {"device": torch.cuda.get_device_name(), "batch": batch, "compute": compute,
            "kernel": layer.describe_path(batch, config.input_h, config.input_w), "time_s": ms * 1e-3,
            "useful_gmacs": macs / (ms * 1e-3) / 1e9}


def run_benchmark_gpu(segconv, configs, options=None, batch: int = 64, compute: str = "fp32"):
    """segconv.bench.run_benchmark with the segregated engine on the GPU (route()), plus a "gpu"
    object per layer record; the reference's report schema otherwise unchanged (emit_report, the
    CLI and the service consume it as is)."""
    route(segconv)
    options = options or segconv.bench.RunOptions()
    report = segconv.bench.run_benchmark(list(configs), options)
    for index, (config, rec) in enumerate(zip(configs, report.layers)):
        if rec.get("error") is None:
            rec["gpu"] = gpu_record(config, options.seed, index, batch, compute)
    return report
