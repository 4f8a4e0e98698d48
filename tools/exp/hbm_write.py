"""HBM write-only / read-only / copy bandwidth at l7-like sizes (torch kernels)."""
import torch
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(it):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best
y = torch.empty(256 * 64 * 256 * 256, dtype=torch.bfloat16, device="cuda")
x = torch.empty(256 * 64 * 128 * 128, dtype=torch.bfloat16, device="cuda")
x.fill_(1)
ms = t(lambda: y.fill_(3))
print(f"fill 2.15 GB: {ms:.3f} ms {y.numel()*2/ms/1e6:.0f} GB/s")
ms = t(lambda: y.zero_())
print(f"zero 2.15 GB: {ms:.3f} ms {y.numel()*2/ms/1e6:.0f} GB/s")
ms = t(lambda: x.sum())
print(f"sum 0.54 GB: {ms:.3f} ms {x.numel()*2/ms/1e6:.0f} GB/s")
y2 = y[: x.numel()]
ms = t(lambda: y2.copy_(x))
print(f"copy 0.54 GB: {ms:.3f} ms {2*x.numel()*2/ms/1e6:.0f} GB/s")
# 20/80 read/write mix: repeat_interleave-like expand (read x once, write 4x)
yv = y.view(256, 64, 128, 2, 128, 2)
xv = x.view(256, 64, 128, 1, 128, 1).expand(256, 64, 128, 2, 128, 2)
ms = t(lambda: yv.copy_(xv))
print(f"nearest-upsample copy 0.54 GB read + 2.15 GB write: {ms:.3f} ms {(x.numel()*2+y.numel()*2)/ms/1e6:.0f} GB/s")
