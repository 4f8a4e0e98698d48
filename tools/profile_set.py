"""One forward of each listed layer (for an ncu --set full capture of every kernel the bench
reports), after an untimed warm-up of all of them:

    python tools/profile_set.py ebgan_l7:fp32:256 ds512_k5:fp32:64 dcgan_l2:bf16:256 ...

Each spec is name:dtype:batch (name from bench.py's layer tables). The script prints the kernel
family each layer dispatches to, in launch order; before each measured layer it launches a
one-element unit_floats kernel as a marker, so a capture filtered with
-k 'regex:unit_floats|direct_kernel|igemm|scatter|absmax|nchw_to_nhwc' splits into layers
(tools/ncu_summary.py).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_20493_b200 as P  # noqa: E402
from paper_2502_20493_b200.synth import device_unit_floats  # noqa: E402


def main():
    table = {c[0]: c for c in bench.EBGAN + bench.DCGAN + bench.DATASET + bench.MNIST}
    runs = []
    for spec in sys.argv[1:]:
        name, dtype, batch = spec.split(":")
        _, h, w, ci, n, co, pad = table[name]
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        bank = device_unit_floats((ci, co, n, n), 5, dtype=torch.float32)
        layer = P.prepare_layer(bank, pad, compute=dtype)
        x = device_unit_floats((int(batch), ci, h, w), 7, dtype=tdt)
        y = torch.empty((int(batch), co) + layer.output_shape(h, w), dtype=tdt, device="cuda")
        runs.append((spec, layer, x, y))
    for _, layer, x, y in runs:  # warm-up
        layer.forward(x, out=y)
    torch.cuda.synchronize()
    for spec, layer, x, y in runs:
        # a one-element unit_floats launch marks where each layer's launches start (include
        # "unit_floats" in ncu's -k filter; tools/ncu_summary.py splits on it)
        device_unit_floats((1,), 0)
        print(f"{spec}: {layer.describe_path(x.shape[0], x.shape[2], x.shape[3])}", flush=True)
        layer.forward(x, out=y)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
