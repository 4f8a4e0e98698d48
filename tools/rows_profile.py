"""Role cycle counters of the K3b kernel (CTA 0) on EB-GAN l7: SEGB200_PROFILE=1."""
import ctypes, os, sys
os.environ["SEGB200_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_20493_b200 as P
from paper_2502_20493_b200 import _lib
from paper_2502_20493_b200.synth import device_unit_floats
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "ebgan_l7"
_, h, w, ci, n, co, pad = {c[0]: c for c in bench.EBGAN + bench.DCGAN}[name]
x = device_unit_floats((256, ci, h, w), 7, dtype=torch.bfloat16)
bank = device_unit_floats((ci, co, n, n), 5, dtype=torch.float32)
layer = P.prepare_layer(bank, pad, compute="bf16")
oh, ow = layer.output_shape(h, w)
y = torch.empty((256, co, oh, ow), dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    layer.forward(x, out=y)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
_lib.lib().segb_debug_rows_profile(buf)
v = list(buf)
names = ["mma wait tempty", "mma wait slots", "mma issue", "epi wait tfull", "epi tmem+cvt", "epi tma-issue",
         "loader wait empty", "loader work", "-", "epi bulk wait", "epi sts", "epi fence"]
for k, nm in enumerate(names):
    print(f"{nm:18s} {v[k]:>12d}")
