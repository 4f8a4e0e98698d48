"""Benchmark: useful GMAC/s of the unified segregated transpose convolution on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A step is one forward pass of every layer of the workload over one synthetic batch.
Default workload: the EB-GAN generator layers l2..l7 (reference GAN_SUITE, bench.py:133-138)
at batch 256 per GPU in fp32 -- the reference's own working precision (engines.py:271-291),
checked against the reference's gate rel 1e-5 / abs 1e-6 (test_acceptance.py:31-32) -- the
BASELINE "EB-GAN generator transpose-conv layers, batch 256" configuration. The same layers in
bf16 (bf16 operands, fp32 accumulation, a stated looser gate) are reported beside it under "bf16".

value    useful MACs (analysis.py:46-57 mult_count_segregated x batch, all ranks)
         / device time of the step (CUDA events, max over ranks), inputs resident.
e2e      the same metric through the public API (PreparedLayer.forward) with
         pinned HOST input/output tensors: H2D + compute + D2H inside the region.
roofline dominant kernel (largest share of the step): algorithmic bytes/flops per launch
          / its average event-timed duration vs the measured peaks.
parity   outside the timed region: sampled outputs of the timed step vs the CPU oracle.
cpu_baseline  the reference's own segregated engine (baseline/_ref, unmodified; the oracle port
         if that is not installed), batch-parallel over the host cores, bounded sample.

--gpus N without torchrun re-launches itself under torch.distributed.run (one rank per GPU).
--impl reference times the reference's CPU path alone (rank 0; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # CPU path parallelises over samples (mode ii)

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

METRIC = "useful GMAC/s per transpose-conv layer and % roofline at 1/2/4/8 B200 vs CPU ref"

# (name, in_h, in_w, c_in, kernel_n, c_out, pad) -- reference GAN_SUITE (bench.py:124-139)
EBGAN = [("ebgan_l2", 4, 4, 2048, 4, 1024, 2), ("ebgan_l3", 8, 8, 1024, 4, 512, 2),
         ("ebgan_l4", 16, 16, 512, 4, 256, 2), ("ebgan_l5", 32, 32, 256, 4, 128, 2),
         ("ebgan_l6", 64, 64, 128, 4, 64, 2), ("ebgan_l7", 128, 128, 64, 4, 64, 2)]
DCGAN = [("dcgan_l2", 4, 4, 1024, 4, 512, 2), ("dcgan_l3", 8, 8, 512, 4, 256, 2),
         ("dcgan_l4", 16, 16, 256, 4, 128, 2), ("dcgan_l5", 32, 32, 128, 4, 3, 2)]
DATASET = [("ds224_k3", 224, 224, 3, 3, 1, 2), ("ds224_k4", 224, 224, 3, 4, 1, 2),
           ("ds224_k5", 224, 224, 3, 5, 1, 2), ("ds512_k5", 512, 512, 3, 5, 1, 2),
           ("ds512_k4_c3", 512, 512, 3, 4, 3, 1)]
MNIST = [("mnist_p0", 28, 28, 1, 3, 1, 0), ("mnist_p1", 28, 28, 1, 3, 1, 1), ("mnist_p2", 28, 28, 1, 3, 1, 2)]

# name -> (layers, batch, dtype, scaling): "weak" = batch per GPU, "strong" = total batch split
# over the ranks (BASELINE config 5)
WORKLOADS = {
    "ebgan_b256_fp32": (EBGAN, 256, "fp32", "weak"),
    "ebgan_b256_bf16": (EBGAN, 256, "bf16", "weak"),
    "ebgan_b4096_bf16": (EBGAN, 4096, "bf16", "strong"),
    "ebgan_b4096_fp32": (EBGAN, 4096, "fp32", "strong"),
    "dcgan_b256_bf16": (DCGAN, 256, "bf16", "weak"),
    "dcgan_b256_fp32": (DCGAN, 256, "fp32", "weak"),
    "dcgan_b64_bf16": (DCGAN, 64, "bf16", "weak"),
    "dcgan_b64_fp32": (DCGAN, 64, "fp32", "weak"),
    "dcgan_b1_bf16": (DCGAN, 1, "bf16", "weak"),
    "dcgan_b1_fp32": (DCGAN, 1, "fp32", "weak"),
    "dataset_b64_fp32": (DATASET, 64, "fp32", "weak"),
    "mnist_b64_fp32": (MNIST, 64, "fp32", "weak"),
}
DEFAULT_WORKLOAD = "ebgan_b256_fp32"
# the precision-matched headline carries the same layers in bf16 beside it
COMPANION = {"ebgan_b256_fp32": "ebgan_b256_bf16", "dcgan_b256_fp32": "dcgan_b256_bf16"}


def load_peaks():
    """HBM and bf16 tensor peaks from the driver's MEASURED_PEAKS.json; the tcgen05 kind::tf32 /
    kind::f16 (fp16) MMA ceilings and the FFMA peak from tools/probes/peak_probe.cu on the box
    (profiles/r2_peaks.json)."""
    out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        out.update(hbm_gbs=d["hbm_gbs"], bf16_tflops=d["bf16_tflops"], source="measured (MEASURED_PEAKS.json)")
        # long steps run power-capped (sw_power_cap): the driver's sustained / burst bf16 ratio
        # scales the compute roofs of kernels timed inside the step ("frac_sustained")
        out["sustained_ratio"] = d.get("bf16_tflops_sustained", d["bf16_tflops"]) / d["bf16_tflops"]
    with open(os.path.join(ROOT, "profiles", "r2_peaks.json")) as f:
        p = json.load(f)
    # the FP32 FMA roof of the direct kernel: register-operand FFMA2 (packed, two FMAs per lane), the
    # fastest FMA form with operands in registers (the immediate-operand FFMA peak does not apply)
    out.update(tf32_mma_tflops=p["tf32_mma_tflops"], fp16_mma_tflops=p["fp16_mma_tflops"],
               ffma_tflops=p.get("ffma2_reg_tflops", p["ffma_tflops"]))
    return out


def layer_stats(cfg, batch, dtype):
    """useful MACs and algorithmic bytes of one layer at `batch`."""
    name, h, w, ci, n, co, pad = cfg
    import paper_2502_20493_b200 as P
    spec = P.TransposeConvSpec(h, w, n, pad, ci, co)
    macs = P.mult_count_segregated(spec) * batch  # analysis.py:46-57, the reference's count
    e = 2 if dtype == "bf16" else 4
    oh, ow = P.output_dims(spec)
    nbytes = batch * ci * h * w * e + batch * co * oh * ow * e + ci * co * n * n * e
    return macs, nbytes, (oh, ow)


def compute_roof(kernel: str, peaks: dict):
    """(TFLOP/s, name) of the unit a layer's kernel (segb_describe_path text) computes on."""
    if kernel.startswith("K3"):
        if "3xFP16" in kernel:  # fp32 as three kind::f16 MMAs per product on scaled fp16 hi/lo
            return peaks["fp16_mma_tflops"] / 3.0, "tensor (3xFP16: fp16 MMA ceiling / 3, measured)"
        if "3xTF32" in kernel:  # three kind::tf32 MMAs per product
            return peaks["tf32_mma_tflops"] / 3.0, "tensor (3xTF32: tf32 MMA ceiling / 3, measured)"
        return peaks["bf16_tflops"], "tensor (bf16, MEASURED_PEAKS)"
    return peaks["ffma_tflops"], "fp32 FMA (register-operand FFMA2, measured)"


# ---------------------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md "clocks" line)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.thread = None

    def wait_first(self, timeout_s: float = 5.0):
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout_s:
            time.sleep(0.01)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# the reference's CPU path (cpu_baseline of our arm, and the whole --impl reference arm)

def host_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except (OSError, subprocess.TimeoutExpired):
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:  # numpy without the dict mode
        pass
    return {"cpu_model": model or platform.processor(), "os_cpu_count": os.cpu_count(), "blas": blas,
            "numpy": np.__version__, "python": platform.python_version()}


def _reference_module():
    """The unmodified reference (tools/install_reference.sh -> baseline/_ref), or None."""
    if os.path.isdir(os.path.join(REF_PATH, "segconv")):
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        try:
            import segconv  # noqa: F401
            return segconv
        except ImportError:
            return None
    return None


class ReferenceCPU:
    """The reference's segregated engine on the host: PreparedLayer(bank, P, "segregated")
    .forward(x_j) per sample (engines.py:246-291), inputs from the reference's own generator and
    the harness seed rule (bench.py:299-300; sample j = gen_synthetic(c, h, w, seed + j*c*h*w),
    the batch stream). Layers are prepared and the sample inputs generated once (untimed, as the
    reference harness, bench.py:257-258); `run()` times one pass over every layer's samples.
    mode "ii": ThreadPoolExecutor(os.cpu_count()) over samples with OPENBLAS_NUM_THREADS=1;
    mode "i": the reference default (threads=1, one sample at a time, OpenBLAS's own threads).
    The unmodified reference comes from baseline/_ref (kind "reference"); without it, the oracle
    port of the same engine (kind "port")."""

    def __init__(self, layers, pass_budget_s: float, mode: str = "ii", samples_cap: int = 256):
        from concurrent.futures import ThreadPoolExecutor

        from oracle.segconv_oracle import harness_seeds, mult_count_segregated
        ref = _reference_module()
        self.cores = os.cpu_count() or 1
        self.mode = mode
        if ref is not None:
            from segconv import engines as E
            from segconv import synth as S
            self.kind = "reference"

            def prep(bank, pad):
                return E.prepare_layer(bank, pad, E.ENGINE_SEGREGATED)
            gen_x, gen_bank = S.gen_synthetic, S.gen_kernel_bank
        else:
            from oracle import segconv_oracle as O
            self.kind = "port"

            class _Port:
                def __init__(self, bank, pad):
                    self.bank, self.pad = bank, pad
                    self.prepared = O.prepare_segregated(bank, np.float32)

                def forward(self, x, threads=1):
                    return O.forward_segregated(x, self.bank, self.pad, prepared=self.prepared)
            prep, gen_x, gen_bank = _Port, O.gen_synthetic, O.gen_kernel_bank
        self.pool = ThreadPoolExecutor(self.cores) if mode == "ii" else None
        self.units, parts = [], []
        par = self.cores if mode == "ii" else 1
        for i, (name, h, w, ci, n, co, pad) in enumerate(layers):
            in_seed, bank_seed = harness_seeds(0, i)
            layer = prep(gen_bank(ci, co, n, bank_seed), pad)
            x0 = gen_x(ci, h, w, in_seed)
            layer.forward(x0)  # warm-up
            t0 = time.perf_counter()
            layer.forward(x0)
            one = time.perf_counter() - t0
            s = int(max(1, min(samples_cap, pass_budget_s / len(layers) * par / max(one, 1e-6))))
            if mode == "ii":
                s = max(s, min(self.cores, samples_cap))
            xs = [gen_x(ci, h, w, in_seed + j * ci * h * w) for j in range(s)]
            self.units.append((layer, xs, mult_count_segregated(h, w, n, pad, ci, co) * s))
            parts.append(f"{name}:{s}")
        self.macs = sum(u[2] for u in self.units)
        what = ("the unmodified reference segconv.PreparedLayer(bank, P, 'segregated').forward (baseline/_ref)"
                if self.kind == "reference" else "the oracle port of the reference's segregated engine")
        how = (f"ThreadPool({self.cores}) over samples, OPENBLAS_NUM_THREADS=1 (mode ii)" if mode == "ii" else
               "one sample at a time, threads=1, OpenBLAS default threading (mode i, the reference default)")
        self.sample = (f"fp32 {what}; samples per layer per pass {{{', '.join(parts)}}}; {how}; per-sample cost is "
                       f"batch-independent (extrapolated to the batch)")

    def run(self) -> float:
        """seconds of one timed pass over all layers' samples"""
        t0 = time.perf_counter()
        for layer, xs, _ in self.units:
            if self.pool is not None:
                list(self.pool.map(layer.forward, xs))
            else:
                for x in xs:
                    layer.forward(x)
        return time.perf_counter() - t0

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def reference_cpu(layers, budget_s: float, mode: str = "ii"):
    """cpu_baseline: one timed pass of ReferenceCPU sized to about budget_s seconds."""
    rc = ReferenceCPU(layers, budget_s, mode)
    try:
        dt = rc.run()
    finally:
        rc.close()
    return {"value": rc.macs / dt / 1e9, "unit": "GMAC/s", "cores": rc.cores, "kind": rc.kind, "mode": mode,
            "sample": rc.sample, "seconds": dt}


def reference_cpu_mode_i(workload: str, budget_s: float):
    """Mode (i) needs OpenBLAS's default threading, fixed at numpy import: run it in a child."""
    env = dict(os.environ)
    env.pop("OPENBLAS_NUM_THREADS", None)
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-ref-worker", "--workload", workload,
           "--cpu-budget", str(budget_s)]
    try:
        res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=max(120, 6 * budget_s))
        return json.loads(res.stdout.strip().splitlines()[-1])
    except Exception as e:  # report, do not fail the bench
        return {"error": f"{type(e).__name__}: {e}"}


def reference_transient(cfg):
    """Per-sample transient host memory of the reference's two engines (tracemalloc peak over
    one forward of the oracle port: np.pad + im2col + GEMM per class, engines.py:271-335, and
    upsample + pad + im2col, engines.py:258-269), the reference side of BASELINE config 4."""
    import tracemalloc

    from oracle import segconv_oracle as O
    name, h, w, ci, n, co, pad = cfg
    in_seed, bank_seed = O.harness_seeds(0, 0)
    x = O.gen_synthetic(ci, h, w, in_seed)
    bank = O.gen_kernel_bank(ci, co, n, bank_seed)
    out = {}
    prep_seg = O.prepare_segregated(bank, np.float32)
    prep_ref = np.ascontiguousarray(bank.transpose(1, 0, 2, 3).reshape(co, -1))
    for key, fn, prep in (("reference_seg_transient_bytes", O.forward_segregated, prep_seg),
                          ("reference_ref_transient_bytes", O.forward_reference, prep_ref)):
        tracemalloc.start()
        y = fn(x, bank, pad, prepared=prep)
        _, peak = tracemalloc.get_traced_memory()
        tracemalloc.stop()
        out[key] = int(peak - y.nbytes)
        del y
    return out


def run_reference(args, rank):
    """--impl reference: the reference's own CPU implementation of the path (the unmodified
    package in baseline/_ref), timed on the host cores; each step is one pass over a bounded
    sample of the workload, sized so that warm-up + steps take about three minutes (rank 0)."""
    if rank != 0:
        return 0
    layers, batch, dtype, scaling = WORKLOADS[args.workload]
    per_pass = float(min(args.ref_step_budget, max(0.5, 180.0 / max(1, args.steps + args.warmup))))
    rc = ReferenceCPU(layers, per_pass, mode="ii")
    try:
        for _ in range(args.warmup):
            rc.run()
        secs = [rc.run() for _ in range(args.steps)]
    finally:
        rc.close()
    dt = float(np.median(secs))
    value = rc.macs / dt / 1e9
    mode_i = reference_cpu_mode_i(args.workload, budget_s=min(20.0, 4 * per_pass))
    out = {"metric": METRIC, "value": value, "unit": "GMAC/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": scaling, "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (reference splitmix64 generator)",
           "config": {"workload": args.workload, "batch_per_gpu": batch, "layers": [c[0] for c in layers]},
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": "GMAC/s", "cores": rc.cores, "kind": rc.kind,
                            "sample": rc.sample + f"; median pass of {args.steps} steps",
                            "mode_i": mode_i, "host": host_info()},
           "e2e": {"value": value, "unit": "GMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# our arm

def pin_to_gpu_numa_node(local_rank: int):
    """Bind this rank's host threads to the CPUs local to its GPU (first-touch NUMA placement of
    the pinned e2e buffers). Returns the previous affinity (or None)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1}
        prev = os.sched_getaffinity(0)
        cpus &= prev
        if cpus:
            os.sched_setaffinity(0, cpus)
            return prev
    except Exception:
        pass
    return None


def _max_over_ranks(v, world, dev):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device="cpu" if dist.get_backend() == "gloo" else dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def parity_check(state, dtype, samples_per_layer: int = 4):
    """Outside the timed region: sampled outputs of the timed step against the fp64 CPU oracle
    (the unified rule, engines.py:271-291). Samples 0, B-1 and seeded random ones, all channels.
    fp32: the reference's gate rel 1e-5 / abs 1e-6 (test_acceptance.py:31-32); bf16: the stated
    bf16 gate on bf16-rounded inputs: rel 2^-7, abs 1e-3 * max|ref|."""
    from oracle import segconv_oracle as O
    rows = []
    for s in state:
        b = s["x"].shape[0]
        rng = np.random.default_rng(1234)
        idx = sorted({0, b - 1} | set(int(v) for v in rng.integers(0, b, max(0, samples_per_layer - 2))))
        bank = s["bank"].double().cpu().numpy()
        if dtype == "bf16":
            bank = O.bf16_round(bank.astype(np.float32)).astype(np.float64)
        worst_rel = worst_abs = 0.0
        ok = True
        for j in idx:
            xj = s["x"][j].float().cpu().numpy().astype(np.float64)
            yj = s["y"][j].float().cpu().numpy()
            ref = O.forward_segregated(xj, bank, s["cfg"][6])
            if dtype == "bf16":
                rep = O.compare(yj, ref, 2.0 ** -7, 1e-3 * float(np.abs(ref).max()))
            else:
                rep = O.compare(yj, ref, 1e-5, 1e-6)
            ok &= rep["passed"]
            worst_rel = max(worst_rel, rep["max_rel_diff"])
            worst_abs = max(worst_abs, rep["max_abs_diff"])
        rows.append({"name": s["name"], "samples": idx, "max_rel": worst_rel, "max_abs": worst_abs, "passed": ok})
    gate = ("rel 1e-5 / abs 1e-6 vs the fp64 oracle (the reference's fp32 gate)" if dtype != "bf16" else
            "rel 2^-7 / abs 1e-3*max|ref| vs the fp64 oracle on bf16-rounded inputs")
    return {"passed": all(r["passed"] for r in rows), "gate": gate, "layers": rows}


def measure(args, workload, rank, world, local_rank, with_e2e=True, with_memory=True, with_parity=True):
    """Prepare, warm up, time `args.steps` steps of `workload` on this rank; return the pieces of
    the JSON line (every rank returns; the caller prints on rank 0)."""
    import torch
    import torch.distributed as dist

    import paper_2502_20493_b200 as P
    from paper_2502_20493_b200 import _lib
    from paper_2502_20493_b200.parallel import shard_range
    from paper_2502_20493_b200.synth import device_unit_floats, harness_seeds

    layers, batch, dtype, scaling = WORKLOADS[workload]
    if args.batch:
        batch = args.batch
    if scaling == "strong":  # BASELINE config 5: one total batch split over the ranks
        b0, b1 = shard_range(batch, world, rank)
    else:                    # batch per GPU
        b0, b1 = rank * batch, (rank + 1) * batch
    local = b1 - b0
    dev = torch.device("cuda", local_rank)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    stream = torch.cuda.current_stream()
    peaks = load_peaks()

    state = []
    for i, cfg in enumerate(layers):
        name, h, w, ci, n, co, pad = cfg
        in_seed, bank_seed = harness_seeds(0, i)
        bank = device_unit_floats((ci, co, n, n), bank_seed, dtype=torch.float32, device=dev)
        layer = P.prepare_layer(bank, pad, compute=dtype)
        # rank r owns samples [b0, b1) of the batch stream
        x = device_unit_floats((local, ci, h, w), in_seed + b0 * ci * h * w, dtype=tdt, device=dev)
        macs, nbytes, (oh, ow) = layer_stats(cfg, local, dtype)
        y = torch.empty((local, co, oh, ow), dtype=tdt, device=dev)
        state.append({"name": name, "cfg": cfg, "layer": layer, "x": x, "y": y, "macs": macs, "bytes": nbytes,
                      "bank": bank, "path": layer.select_path(_lib.BF16 if dtype == "bf16" else _lib.F32, local, h, w),
                      "kernel": layer.describe_path(local, h, w), "flops": 2 * macs})
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    sampler.wait_first()
    for _ in range(max(args.warmup, 3)):
        for s in state:
            s["layer"].forward(s["x"], out=s["y"])
    torch.cuda.synchronize()

    mem_rows = []
    if with_memory:
        for s in state:
            mem_rows.append({"name": s["name"], "path": s["path"],
                             "workspace_bytes": s["layer"].workspace_bytes(local, s["cfg"][1], s["cfg"][2]),
                             "io_bytes": s["x"].numel() * s["x"].element_size() + s["y"].numel() * s["y"].element_size(),
                             "upsampled_buffer_bytes_avoided": local * P.memory_savings_bytes(
                                 s["cfg"][1], s["cfg"][2], s["cfg"][6], s["cfg"][3],
                                 element_bytes=s["x"].element_size())})

    # CUDA graphs instead of a tracing compiler: the whole step (every layer's public-API
    # forward) is captured once and replayed as one graph per timed step; the per-layer breakdown
    # replays one graph per layer with events between them (after every fourth timed step)
    graphs, step_graph, launches_per_step = [], None, 0
    if not args.no_graph:
        for s in state:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                s["layer"].forward(s["x"], out=s["y"])
            graphs.append(g)
        step_graph = torch.cuda.CUDAGraph()
        c0 = _lib.launch_count()
        with torch.cuda.graph(step_graph):
            for s in state:
                s["layer"].forward(s["x"], out=s["y"])
        launches_per_step = _lib.launch_count() - c0
        torch.cuda.synchronize()
        for g in graphs:
            g.replay()
        step_graph.replay()
        torch.cuda.synchronize()

    def step(events=None):
        for j, s in enumerate(state):
            if graphs:
                graphs[j].replay()
            else:
                s["layer"].forward(s["x"], out=s["y"])
            if events is not None:
                events[j].record(stream)

    per_layer = [[] for _ in state]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_traffic = sum(s["bytes"] for s in state)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if step_traffic < (252 << 20) else None
    launches0 = _lib.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    evs = [[torch.cuda.Event(enable_timing=True) for _ in state] for _ in range(args.steps)]
    if step_graph is not None:
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        bks = list(range(0, args.steps, 4))
        bstarts = [torch.cuda.Event(enable_timing=True) for _ in bks]
        for k in range(args.steps):
            if flush is not None:
                flush.fill_(k & 0xFF)
            starts[k].record(stream)
            step_graph.replay()
            ends[k].record(stream)
            if k % 4 == 0:
                if flush is not None:
                    flush.fill_((k + 1) & 0xFF)
                bstarts[k // 4].record(stream)
                step(evs[k // 4])
        torch.cuda.synchronize()
        launches = (_lib.launch_count() - launches0) + launches_per_step * args.steps
        if world > 1:
            dist.barrier()
        clocks = sampler.stop()
        ms = float(np.mean([starts[k].elapsed_time(ends[k]) for k in range(args.steps)]))
        starts, nbreak = bstarts, len(bks)
    else:
        for k in range(args.steps):
            if flush is not None:
                flush.fill_(k & 0xFF)
            starts[k].record(stream)
            step(evs[k])
        torch.cuda.synchronize()
        launches = _lib.launch_count() - launches0
        if world > 1:
            dist.barrier()
        clocks = sampler.stop()
        ms = float(np.mean([starts[k].elapsed_time(evs[k][-1]) for k in range(args.steps)]))
        nbreak = args.steps
    for k in range(nbreak):
        prev = starts[k]
        for j in range(len(state)):
            per_layer[j].append(prev.elapsed_time(evs[k][j]))
            prev = evs[k][j]
    ms = _max_over_ranks(ms, world, dev)

    step_macs_local = sum(s["macs"] for s in state)
    total_macs = sum(layer_stats(c, batch if scaling == "strong" else batch * world, dtype)[0] for c in layers)
    value = total_macs / (ms * 1e-3) / 1e9

    capped = bool(clocks) and "sw_power_cap" in (clocks.get("reasons") or [])
    layer_rows = []
    for j, s in enumerate(state):
        lms = float(np.mean(per_layer[j]))
        cpeak, cname = compute_roof(s["kernel"], peaks)
        t_comp = s["flops"] / (cpeak * 1e12)
        t_hbm = s["bytes"] / (peaks["hbm_gbs"] * 1e9)
        bound = "tensor" if (t_comp > t_hbm and s["path"] == "igemm") else ("ffma" if t_comp > t_hbm else "hbm")
        if bound != "hbm":
            achieved, peak, unit = s["flops"] / (lms * 1e-3) / 1e12, cpeak, "TFLOP/s"
        else:
            achieved, peak, unit = s["bytes"] / (lms * 1e-3) / 1e9, peaks["hbm_gbs"], "GB/s"
        layer_rows.append({"name": s["name"], "path": s["path"], "kernel": s["kernel"], "ms": lms,
                           "gmacs": s["macs"] / (lms * 1e-3) / 1e9, "bound": bound, "peak_name": cname,
                           "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                           # against the driver's sustained peak, for runs that hit the power cap
                           "frac_sustained": (achieved / (peak * peaks.get("sustained_ratio", 1.0)) if bound != "hbm"
                                              else achieved / peak) if capped else None,
                           "alg_bytes": s["bytes"], "flops": s["flops"]})
    dom = max(layer_rows, key=lambda r: r["ms"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(workload, {}).get(dom["name"])
    roofline = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["frac"], "traffic": traffic, "kernel": f"{dom['name']}: {dom['kernel']}",
                "share_of_step": dom["ms"] / ms, "peak_source": dom["peak_name"] if dom["bound"] != "hbm"
                else peaks["source"]}

    parity = parity_check(state, dtype) if (with_parity and rank == 0) else None

    e2e = None
    if with_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        hx = [s["x"].cpu().pin_memory() for s in state]
        hy = [torch.empty(s["y"].shape, dtype=tdt).pin_memory() for s in state]
        h2d = sum(t.numel() * t.element_size() for t in hx)
        d2h = sum(t.numel() * t.element_size() for t in hy)

        def e2e_step():
            # every layer through the public API with host tensors; each layer's D2H copies stay in
            # flight (non_blocking) while the next layer's input copies and kernels run, and the step
            # ends with the stream ordered after all of them (wait_host_copies), so the closing event
            # counts every byte
            for s, xi, yi in zip(state, hx, hy):
                s["layer"].forward(xi, out=yi, non_blocking=True)
            P.wait_host_copies(dev)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = _max_over_ranks(e0.elapsed_time(e1) / e2e_steps, world, dev)
        e2e = {"value": total_macs / (ems * 1e-3) / 1e9, "unit": "GMAC/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ems,
               "steps": e2e_steps, "api": "PreparedLayer.forward(pinned host tensor, out=pinned host tensor)"}
        chains = all(a["cfg"][5] == b["cfg"][3] and tuple(a["y"].shape[2:]) == tuple(b["x"].shape[2:])
                     for a, b in zip(state, state[1:]))
        if chains and len(state) > 1:
            stack = P.prepare_stack([s["layer"] for s in state])
            sx, sy = hx[0], hy[-1]
            stack.forward(sx, out=sy)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0.record(stream)
            for _ in range(e2e_steps):
                stack.forward(sx, out=sy)
            e1.record(stream)
            torch.cuda.synchronize()
            sms = _max_over_ranks(e0.elapsed_time(e1) / e2e_steps, world, dev)
            e2e["stack"] = {"value": total_macs / (sms * 1e-3) / 1e9, "unit": "GMAC/s", "ms_per_step": sms,
                            "h2d_bytes_per_step": sx.numel() * sx.element_size(),
                            "d2h_bytes_per_step": sy.numel() * sy.element_size(),
                            "api": f"PreparedStack.forward(pinned host tensor, out=pinned host tensor): l2..lN "
                                   f"chained on the device ({stack.inter_dtype} intermediates), one CUDA graph"}
            del stack
        del hx, hy

    res = {"value": value, "ms_per_step": ms, "roofline": roofline, "layers": layer_rows, "parity": parity,
           "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks, "memory": mem_rows, "batch": batch,
           "local_batch": local, "scaling": scaling, "dtype": dtype, "step_macs_local": step_macs_local,
           "step_traffic": step_traffic, "flushed": flush is not None, "graph": not args.no_graph}
    del state, graphs, step_graph
    torch.cuda.empty_cache()
    return res


def run_ours(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    prev_affinity = None if os.environ.get("SEGB200_NO_NUMA_PIN") else pin_to_gpu_numa_node(local_rank)
    wl = args.workload
    layers, batch, dtype, scaling = WORKLOADS[wl]
    big = scaling == "strong"  # config 5: multi-GB host buffers, no e2e leg by default
    r = measure(args, wl, rank, world, local_rank, with_e2e=not (args.no_e2e or big),
                with_memory=True, with_parity=not args.no_parity)
    companion = None
    if COMPANION.get(wl) and not args.no_companion:
        c = measure(args, COMPANION[wl], rank, world, local_rank, with_e2e=not args.no_e2e, with_memory=False,
                    with_parity=not args.no_parity)
        companion = {"workload": COMPANION[wl], "dtype": "bf16", "value": c["value"], "unit": "GMAC/s",
                     "ms_per_step": c["ms_per_step"], "roofline": c["roofline"], "parity": c["parity"],
                     "e2e": c["e2e"], "gpu_launches": c["gpu_launches"], "clocks": c["clocks"],
                     "layers": [{k: row[k] for k in ("name", "kernel", "ms", "gmacs", "bound", "frac", "frac_sustained")}
                                for row in c["layers"]]}
    if rank != 0:
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        if prev_affinity:
            os.sched_setaffinity(0, prev_affinity)
        cpu = reference_cpu(layers, budget_s=args.cpu_budget, mode="ii")
        cpu["host"] = host_info()
        if not args.no_memory_reference:
            for row, cfg in zip(r["memory"], layers):
                row.update(reference_transient(cfg))
    flush_note = (f"L2 flushed before every step (256 MB write, untimed); {r['step_traffic'] / 1e6:.1f} MB "
                  f"algorithmic traffic per step" if r["flushed"] else
                  f"inputs larger than L2: {r['step_traffic'] / 1e9:.2f} GB algorithmic traffic per step vs "
                  f"126 MB L2 (no explicit flush)")
    out = {"metric": METRIC, "value": r["value"], "unit": "GMAC/s", "n_gpus": world, "steps": args.steps,
           "warmup": max(args.warmup, 3), "ms_per_step": r["ms_per_step"], "higher_is_better": True,
           "scaling": scaling, "vs_baseline": None, "dtype": "bf16" if dtype == "bf16" else "f32",
           "data": "synthetic (reference splitmix64 generator, produced on device)",
           "config": {"workload": wl, "batch_per_gpu": r["local_batch"], "total_batch": r["batch"] if scaling ==
                      "strong" else r["batch"] * world, "layers": [c[0] for c in layers],
                      "precision": ("fp32 in/out; tensor-core layers as 3xFP16 (power-of-two scaled fp16 hi/lo "
                                    "planes, hi*hi + hi*lo + lo*hi in fp32, unscaled exactly), direct layers FFMA; "
                                    "gate rel 1e-5 / abs 1e-6" if dtype == "fp32" else
                                    "bf16 operands, fp32 accumulation, bf16 out"),
                      "launch": "eager" if args.no_graph else
                      "one CUDA graph per step (per-layer graphs for the layer breakdown)", "l2": flush_note},
           "parity": r["parity"], "roofline": r["roofline"], "cpu_baseline": cpu, "e2e": r["e2e"],
           "gpu_launches": r["gpu_launches"], "clocks": r["clocks"], "layers": r["layers"],
           "memory": {"note": "workspace = device bytes segb_forward_ws takes beyond x, y and the prepared "
                              "weights (segb_forward_workspace_bytes); reference_*_transient = tracemalloc peak of "
                              "one sample through the CPU oracle port of the reference engines; "
                              "upsampled_buffer_bytes_avoided = memory_savings_bytes (analysis.py:60-82) x batch",
                      "layers": r["memory"]}}
    if companion is not None:
        out["bf16"] = companion
    print(json.dumps(out), flush=True)
    return 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager API calls instead of CUDA-graph replays")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-companion", action="store_true", help="skip the bf16 line beside the fp32 headline")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-step-budget", type=float, default=8.0,
                    help="--impl reference: host seconds of reference work per step")
    ap.add_argument("--no-memory-reference", action="store_true",
                    help="skip the tracemalloc pass over the CPU oracle (reference memory footprint)")
    ap.add_argument("--cpu-ref-worker", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()

    if args.cpu_ref_worker:  # child of reference_cpu_mode_i: OpenBLAS default threading
        layers = WORKLOADS[args.workload][0]
        print(json.dumps(reference_cpu(layers, budget_s=args.cpu_budget, mode="i")), flush=True)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one rank per GPU: re-launch under torch.distributed.run on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank)
    # SEGB200_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo -- a functional check of the N > 1
    # path (sharding, barriers, max over ranks, the JSON line) on a one-GPU machine; not a number
    share = world > 1 and os.environ.get("SEGB200_BENCH_SHARE_GPU") == "1"
    dev_rank = 0 if share else local_rank
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")       # the init log shows nranks / the transport
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(dev_rank)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, dev_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
