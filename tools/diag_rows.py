
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_20493_b200 as P
from oracle import segconv_oracle as O
from paper_2502_20493_b200.synth import device_unit_floats
h=w=128; ci=64; n=4; co=64; pad=2; b=1
x = device_unit_floats((b, ci, h, w), 3, dtype=torch.bfloat16)
bank = O.gen_kernel_bank(ci, co, n, 4)
ref = O.forward_segregated_batch(x.float().cpu().numpy().astype(np.float64), O.bf16_round(bank).astype(np.float64), pad)
layer = P.prepare_layer(bank, pad, compute="bf16")
y = layer.forward(x, path="igemm", out_dtype=torch.float32).cpu().numpy()
print("boff", os.environ.get("SEGB200_ROWS_BOFF"), O.compare(y, ref, 1e-4, 1e-5), flush=True)
d = np.abs(y - ref)[0]
print("bad fraction per class (r,s):", [[float((d[:, r::2, s::2] > 1e-3 * np.abs(ref).max()).mean()) for s in (0, 1)] for r in (0, 1)])
