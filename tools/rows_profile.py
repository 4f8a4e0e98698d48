"""Role cycle counters of the K3b kernel (CTA 0; library built with -D SEGB_ROWS_PROFILE, run with
SEGB200_PROFILE=1): python tools/rows_profile.py [layer] [bf16|fp32]"""
import ctypes, os, sys
os.environ["SEGB200_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_20493_b200 as P
from paper_2502_20493_b200 import _lib
from paper_2502_20493_b200.synth import device_unit_floats
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "ebgan_l7"
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
_, h, w, ci, n, co, pad = {c[0]: c for c in bench.EBGAN + bench.DCGAN}[name]
x = device_unit_floats((256, ci, h, w), 7, dtype=tdt)
bank = device_unit_floats((ci, co, n, n), 5, dtype=torch.float32)
layer = P.prepare_layer(bank, pad, compute=dtype)
oh, ow = layer.output_shape(h, w)
y = torch.empty((256, co, oh, ow), dtype=tdt, device="cuda")
for _ in range(2):
    layer.forward(x, out=y)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
_lib.lib().segb_debug_rows_profile(buf)
v = list(buf)
names = ["mma wait tempty", "mma wait slots", "mma issue", "epi wait tfull", "epi work", "epi tma-issue",
         "loader wait empty", "loader work", "-", "epi bulk wait", "epi sts", "epi fence",
         "loader convert+sts", "loader arrive", "loader fence"]
for k, nm in enumerate(names):
    print(f"{nm:18s} {v[k]:>12d}")
