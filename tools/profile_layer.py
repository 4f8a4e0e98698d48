"""Run one benchmark layer's forward a few times (for ncu captures and quick timing).

    python tools/profile_layer.py ebgan_l7 [--batch 256] [--iters 3] [--dtype bf16] [--path auto]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_20493_b200 as P  # noqa: E402
from paper_2502_20493_b200.synth import device_unit_floats  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("layer")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--path", default="auto")
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays (no host gaps)")
    a = ap.parse_args()
    cfg = {c[0]: c for c in bench.EBGAN + bench.DCGAN + bench.DATASET + bench.MNIST}[a.layer]
    name, h, w, ci, n, co, pad = cfg
    tdt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    bank = device_unit_floats((ci, co, n, n), 5, dtype=torch.float32)
    layer = P.prepare_layer(bank, pad, compute=a.dtype)
    x = device_unit_floats((a.batch, ci, h, w), 7, dtype=tdt)
    oh, ow = layer.output_shape(h, w)
    y = torch.empty((a.batch, co, oh, ow), dtype=tdt, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run = lambda: layer.forward(x, out=y, path=a.path)  # noqa: E731
    if a.graph:  # replay a captured graph: no host launch gaps inside the timed region
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            layer.forward(x, out=y, path=a.path)
        run = g.replay
    for i in range(a.iters):
        s.record()
        run()
        e.record()
        torch.cuda.synchronize()
        print(f"{name} iter {i}: {s.elapsed_time(e):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
