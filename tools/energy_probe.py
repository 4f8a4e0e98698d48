"""Steady-state time, SM clock and board power of each layer's forward when it runs back to back
for a few seconds (the fp32 EB-GAN step runs under sw_power_cap, so energy per forward, not the
burst time, is what its step time follows):

    python tools/energy_probe.py [fp32|bf16] [seconds]
"""
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_20493_b200 as P  # noqa: E402
from paper_2502_20493_b200.synth import device_unit_floats  # noqa: E402


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                            "-i", "0"], capture_output=True, text=True)
        try:
            p, c = r.stdout.strip().split(",")
            out.append((float(p), float(c)))
        except ValueError:
            pass
        time.sleep(0.05)


def main():
    dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    for name, h, w, ci, n, co, pad in bench.EBGAN:
        layer = P.prepare_layer(device_unit_floats((ci, co, n, n), 5), pad, compute=dtype)
        x = device_unit_floats((256, ci, h, w), 7, dtype=tdt)
        y = torch.empty((256, co) + layer.output_shape(h, w), dtype=tdt, device="cuda")
        layer.forward(x, out=y)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                layer.forward(x, out=y)
        g.replay()
        torch.cuda.synchronize()
        stop, samples = threading.Event(), []
        th = threading.Thread(target=sample, args=(stop, samples))
        t_end = time.time() + secs
        reps = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        th.start()
        time.sleep(0.2)
        e0.record()
        while time.time() < t_end:
            for _ in range(5):
                g.replay()
            reps += 50
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / reps
        tail = samples[len(samples) // 3:]
        pw = sum(p for p, _ in tail) / max(1, len(tail))
        ck = sorted(c for _, c in tail)[len(tail) // 2] if tail else 0
        print(f"{name} {dtype}: {ms:.3f} ms/forward, {pw:.0f} W, SM {ck:.0f} MHz, {pw * ms:.0f} mJ/forward",
              flush=True)


if __name__ == "__main__":
    main()
