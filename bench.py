"""Benchmark: useful GMAC/s of the unified segregated transpose convolution on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A step is one forward pass of every layer of the workload over one synthetic
batch (per GPU; weak scaling across ranks: batch sharding needs no collective).
Default workload: the EB-GAN generator layers l2..l7 (reference GAN_SUITE,
bench.py:133-138) at batch 256 per GPU in bf16 (fp32 accumulation), the
BASELINE "EB-GAN generator transpose-conv layers, batch 256" configuration.

value    useful MACs (analysis.py:46-57 mult_count_segregated x batch, all ranks)
         / device time of the step (CUDA events, max over ranks), inputs resident.
e2e      the same metric through the public API (PreparedLayer.forward) with
         pinned HOST input/output tensors: H2D + compute + D2H inside the region.
roofline dominant kernel (largest share of the step): algorithmic bytes/flops per
         launch / its average event-timed duration vs MEASURED_PEAKS.
cpu_baseline  the CPU oracle port of the reference's segregated engine (numpy /
         OpenBLAS, batch-parallel over host threads) on a bounded sample, rank 0, N=1.

--impl reference times that CPU path alone (rank 0; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # CPU path parallelises over samples

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

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

WORKLOADS = {
    "ebgan_b256_bf16": (EBGAN, 256, "bf16"),
    "ebgan_b256_fp32": (EBGAN, 256, "fp32"),
    "dcgan_b256_bf16": (DCGAN, 256, "bf16"),
    "dcgan_b256_fp32": (DCGAN, 256, "fp32"),
    "dataset_b64_fp32": (DATASET, 64, "fp32"),
    "mnist_b64_fp32": (MNIST, 64, "fp32"),
}
DEFAULT_WORKLOAD = "ebgan_b256_bf16"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


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
        """Block until nvidia-smi has produced its first sample (it takes a moment to start)."""
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

def cpu_baseline(layers, dtype, budget_s: float = 20.0):
    """The reference's segregated CPU engine (oracle port: numpy im2col + OpenBLAS GEMM per
    parity class, engines.py:271-335), batch-parallel over host threads, bounded sample."""
    from oracle import segconv_oracle as O
    cores = os.cpu_count() or 1
    total_macs, total_s, parts = 0, 0.0, []
    for i, (name, h, w, ci, n, co, pad) in enumerate(layers):
        in_seed, bank_seed = O.harness_seeds(0, i)
        bank = O.gen_kernel_bank(ci, co, n, bank_seed)
        per = O.mult_count_segregated(h, w, n, pad, ci, co)
        # one warm-up sample, then `cores` samples (at least 1) within the time budget
        x1 = O.gen_synthetic(ci, h, w, in_seed)
        t0 = time.perf_counter()
        O.forward_segregated(x1, bank, pad)
        one = time.perf_counter() - t0
        budget_layer = budget_s / len(layers)
        s = int(max(1, min(256, budget_layer * cores / max(one, 1e-6))))
        xs = O.unit_floats(s * ci * h * w, in_seed).reshape(s, ci, h, w)
        t0 = time.perf_counter()
        O.forward_segregated_batch(xs, bank, pad, workers=cores)
        dt = time.perf_counter() - t0
        total_macs += per * s
        total_s += dt
        parts.append(f"{name}:{s}")
    return {"value": total_macs / total_s / 1e9, "unit": "GMAC/s", "cores": cores, "kind": "port",
            "sample": f"fp32 numpy/OpenBLAS segregated engine, samples per layer {{{', '.join(parts)}}}, "
                      f"ThreadPool({cores}) over samples, OPENBLAS_NUM_THREADS=1; per-sample cost is "
                      f"batch-independent (extrapolated to batch)",
            "seconds": total_s}


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
    # weights are laid out once per weight tensor outside the forward (engines.py:232-244)
    prep_seg = O.prepare_segregated(bank, np.float32)
    prep_ref = np.ascontiguousarray(bank.transpose(1, 0, 2, 3).reshape(co, -1))
    for key, fn, prep in (("reference_seg_transient_bytes", O.forward_segregated, prep_seg),
                          ("reference_ref_transient_bytes", O.forward_reference, prep_ref)):
        tracemalloc.start()
        y = fn(x, bank, pad, prepared=prep)
        _, peak = tracemalloc.get_traced_memory()
        tracemalloc.stop()
        out[key] = int(peak - y.nbytes)  # transient beyond the returned output
        del y
    return out


def run_reference(args, rank):
    layers, batch, dtype = WORKLOADS[args.workload]
    if rank != 0:
        return 0
    from oracle import segconv_oracle as O
    cores = os.cpu_count() or 1
    s = max(1, min(cores, 16))
    prepared = []
    for i, (name, h, w, ci, n, co, pad) in enumerate(layers):
        in_seed, bank_seed = O.harness_seeds(0, i)
        prepared.append((O.unit_floats(s * ci * h * w, in_seed).reshape(s, ci, h, w),
                         O.gen_kernel_bank(ci, co, n, bank_seed), pad,
                         O.mult_count_segregated(h, w, n, pad, ci, co) * s))
    macs = sum(p[3] for p in prepared)

    def step():
        for x, bank, pad, _ in prepared:
            O.forward_segregated_batch(x, bank, pad, workers=cores)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = macs / dt / 1e9
    sample = (f"{s} samples per layer per step (bounded sample of batch {batch}), fp32 numpy/OpenBLAS "
              f"oracle port of the reference segregated engine, ThreadPool({cores}) over samples")
    out = {"metric": METRIC, "value": value, "unit": "GMAC/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference splitmix64 generator)",
           "config": {"workload": args.workload, "batch_per_gpu": batch, "layers": [c[0] for c in layers]},
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": "GMAC/s", "cores": cores, "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": "GMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def pin_to_gpu_numa_node(local_rank: int):
    """Bind this rank's host threads to the CPUs nvidia-smi reports as local to its GPU, so the
    pinned host buffers of the e2e leg are allocated on the GPU's NUMA node (first touch) and
    PCIe copies do not cross the socket interconnect. Returns the previous affinity (or None)."""
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
    except Exception:  # no NVML or no affinity info: leave the binding alone
        pass
    return None


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2502_20493_b200 as P
    from paper_2502_20493_b200 import _lib
    from paper_2502_20493_b200.synth import device_unit_floats, harness_seeds

    layers, batch, dtype = WORKLOADS[args.workload]
    if args.batch:
        batch = args.batch
    torch.cuda.set_device(local_rank)
    prev_affinity = None if os.environ.get("SEGB200_NO_NUMA_PIN") else pin_to_gpu_numa_node(local_rank)
    dev = torch.device("cuda", local_rank)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    stream = torch.cuda.current_stream()

    # --- prepare (untimed, as the reference harness, bench.py:257-258) ---
    state = []
    for i, cfg in enumerate(layers):
        name, h, w, ci, n, co, pad = cfg
        in_seed, bank_seed = harness_seeds(0, i)
        bank = device_unit_floats((ci, co, n, n), bank_seed, dtype=torch.float32, device=dev)
        layer = P.prepare_layer(bank, pad, compute=dtype)
        # rank r owns samples [r*batch, (r+1)*batch) of the batch stream
        x = device_unit_floats((batch, ci, h, w), in_seed + rank * batch * ci * h * w, dtype=tdt, device=dev)
        macs, nbytes, (oh, ow) = layer_stats(cfg, batch, dtype)
        y = torch.empty((batch, co, oh, ow), dtype=tdt, device=dev)
        state.append({"name": name, "cfg": cfg, "layer": layer, "x": x, "y": y, "macs": macs, "bytes": nbytes,
                      "path": layer.select_path(_lib.BF16 if dtype == "bf16" else _lib.F32, batch, h, w),
                      "flops": 2 * macs})
    torch.cuda.synchronize()

    # clocks are sampled from the warm-up on (the GPU is under the same load) through the
    # end of the timed region; nvidia-smi needs a moment to start
    sampler = ClockSampler(local_rank)
    sampler.start()
    sampler.wait_first()
    for _ in range(max(args.warmup, 3)):
        for s in state:
            s["layer"].forward(s["x"], out=s["y"])
    torch.cuda.synchronize()

    # device memory beyond inputs, outputs and prepared weights (BASELINE config 4: memory
    # footprint vs the reference): the forward workspace high-water mark per layer
    mem_rows = []
    for s in state:
        _lib.workspace_high_water(local_rank, reset=True)
        s["layer"].forward(s["x"], out=s["y"])
        torch.cuda.synchronize()
        mem_rows.append({"name": s["name"], "path": s["path"],
                         "workspace_bytes": _lib.workspace_high_water(local_rank),
                         "io_bytes": s["x"].numel() * s["x"].element_size() + s["y"].numel() * s["y"].element_size(),
                         "upsampled_buffer_bytes_avoided": batch * P.memory_savings_bytes(
                             s["cfg"][1], s["cfg"][2], s["cfg"][6], s["cfg"][3], element_bytes=s["x"].element_size())})

    # CUDA graphs instead of a tracing compiler: the whole step (every layer's forward, the
    # public API call) is captured once and replayed as one graph in the timed loop, so it has
    # no Python and one launch per step; the per-layer breakdown comes from a second loop that
    # replays one graph per layer with events between them (outside the graphs).
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
    # L2 hygiene: a step that moves less than 2x the 126 MB L2 is preceded by a 256 MB
    # write (outside the timed span of the step), so every step starts L2-cold
    step_traffic = sum(s["bytes"] for s in state)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if step_traffic < (252 << 20) else None
    launches0 = _lib.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    evs = [[torch.cuda.Event(enable_timing=True) for _ in state] for _ in range(args.steps)]
    if step_graph is not None:
        # the timed steps (one graph replay each, between starts[k] and ends[k]) interleaved
        # with the per-layer breakdown (per-layer graphs, events between them), so both see the
        # same clocks and power state; only the former gives ms_per_step and value
        # (the breakdown follows every 4th timed step: enough samples, little extra sustained load)
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
        launches = (_lib.launch_count() - launches0) + launches_per_step * args.steps  # inside the timed steps
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
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    peaks = load_peaks()
    step_macs = sum(s["macs"] for s in state)
    value = step_macs * world / (ms * 1e-3) / 1e9

    # per-layer roofline: bound = the larger of compute time and HBM time, where the compute
    # peak is the one of the unit the layer runs on: measured bf16 tensor peak (K3/K3b bf16);
    # for 3xTF32 (K3 fp32) the measured bf16 peak / 2 (tf32 rate) / 3 (passes); for the
    # CUDA-core direct kernel the FFMA peak 148 SM x 128 x 2 x 1.965 GHz (theoretical)
    layer_rows = []
    for j, s in enumerate(state):
        lms = float(np.mean(per_layer[j]))
        if s["path"] == "igemm":
            cpeak = peaks["bf16_tflops"] if dtype == "bf16" else peaks["bf16_tflops"] / 6.0
            cname = "tensor"
        else:
            cpeak, cname = 148 * 128 * 2 * 1.965e-3, "fp32_ffma"
        t_comp = s["flops"] / (cpeak * 1e12)
        t_hbm = s["bytes"] / (peaks["hbm_gbs"] * 1e9)
        bound = cname if t_comp > t_hbm else "hbm"
        if bound != "hbm":
            achieved, peak, unit = s["flops"] / (lms * 1e-3) / 1e12, cpeak, "TFLOP/s"
        else:
            achieved, peak, unit = s["bytes"] / (lms * 1e-3) / 1e9, peaks["hbm_gbs"], "GB/s"
        layer_rows.append({"name": s["name"], "path": s["path"], "ms": lms,
                           "gmacs": s["macs"] / (lms * 1e-3) / 1e9, "bound": bound,
                           "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                           "alg_bytes": s["bytes"], "flops": s["flops"]})
    dom = max(layer_rows, key=lambda r: r["ms"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(args.workload, {}).get(dom["name"])
    roofline = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["frac"], "traffic": traffic, "kernel": f"{dom['name']} ({dom['path']})",
                "share_of_step": dom["ms"] / ms, "peak_source": peaks["source"]}

    # --- e2e through the public API with pinned host buffers ---
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        hx = [s["x"].cpu().pin_memory() for s in state]
        hy = [torch.empty(s["y"].shape, dtype=tdt).pin_memory() for s in state]
        h2d = sum(t.numel() * t.element_size() for t in hx)
        d2h = sum(t.numel() * t.element_size() for t in hy)

        def e2e_step():
            for s, xi, yi in zip(state, hx, hy):
                s["layer"].forward(xi, out=yi)

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
        ems = e0.elapsed_time(e1) / e2e_steps
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": step_macs * world / (ems * 1e-3) / 1e9, "unit": "GMAC/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ems,
               "steps": e2e_steps, "api": "PreparedLayer.forward(pinned host tensor, out=pinned host tensor)",
               "host_threads_on_gpu_numa_node": bool(prev_affinity)}
        # the same layers as one device-resident generator stack: only the
        # first layer's input goes up and the last layer's output comes back
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
            sms = e0.elapsed_time(e1) / e2e_steps
            if world > 1:
                t = torch.tensor([sms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                sms = float(t.item())
            e2e["stack"] = {"value": step_macs * world / (sms * 1e-3) / 1e9, "unit": "GMAC/s", "ms_per_step": sms,
                            "h2d_bytes_per_step": sx.numel() * sx.element_size(),
                            "d2h_bytes_per_step": sy.numel() * sy.element_size(),
                            "api": "PreparedStack.forward(pinned host tensor, out=pinned host tensor): "
                                   "l2..lN chained on the device (bf16 intermediates), one CUDA graph"}
            del stack
        del hx, hy

    if rank != 0:
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        if prev_affinity:  # the CPU baseline gets every host core back
            os.sched_setaffinity(0, prev_affinity)
        cpu = cpu_baseline(layers, dtype, budget_s=args.cpu_budget)
        if not args.no_memory_reference:
            for row, cfg in zip(mem_rows, layers):
                row.update(reference_transient(cfg))
    total_traffic = sum(s["bytes"] for s in state)
    out = {"metric": METRIC, "value": value, "unit": "GMAC/s", "n_gpus": world, "steps": args.steps,
           "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16" if dtype == "bf16" else "f32",
           "data": "synthetic (reference splitmix64 generator, produced on device)",
           "config": {"workload": args.workload, "batch_per_gpu": batch, "layers": [s["name"] for s in state],
                      "accumulate": "fp32", "launch": "eager" if args.no_graph else "one CUDA graph per step (per-layer graphs for the layer breakdown)",
                      "l2": (f"inputs larger than L2: {total_traffic / 1e9:.2f} GB algorithmic traffic per "
                             f"step vs 126 MB L2 (no explicit flush)" if flush is None else
                             f"L2 flushed before every step (256 MB write, untimed); {total_traffic / 1e6:.1f} MB "
                             f"algorithmic traffic per step")},
           "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
           "clocks": clocks, "layers": layer_rows,
           "memory": {"note": "workspace = device bytes segb_forward takes beyond x, y and the prepared "
                              "weights (batch of the workload); reference_*_transient = tracemalloc peak of "
                              "one sample through the CPU oracle port of the reference engines; "
                              "upsampled_buffer_bytes_avoided = memory_savings_bytes (analysis.py:60-82) x batch",
                      "layers": mem_rows}}
    print(json.dumps(out), flush=True)
    return 0


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
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-memory-reference", action="store_true",
                    help="skip the tracemalloc pass over the CPU oracle (reference memory footprint)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
