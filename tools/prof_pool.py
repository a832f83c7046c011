"""Time the maxpool forward / backward launches on the ResNet stem shape
(256 x 64 x 112 x 112 bf16 NHWC, 3x3/2/1):  python tools/prof_pool.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_12406_b200 import functional as MF  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.randn(256, 64, 112, 112, device=dev, dtype=torch.bfloat16)
x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
g = torch.randn(256, 64, 56, 56, device=dev, dtype=torch.bfloat16)
g = g.contiguous(memory_format=torch.channels_last)
for _ in range(3):
    y = MF.max_pool2d(x, 3, 2, 1)
    y.backward(g)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
s.record()
for _ in range(reps):
    y = MF.max_pool2d(x, 3, 2, 1)
e.record()
torch.cuda.synchronize()
fwd = s.elapsed_time(e) / reps
s.record()
for _ in range(reps):
    x.grad = None
    y.backward(g, retain_graph=True)
e.record()
torch.cuda.synchronize()
bwd = s.elapsed_time(e) / reps
gb_f = (x.numel() * 2 + y.numel() * 3) / 1e9
gb_b = (g.numel() * 3 + x.numel() * 2) / 1e9
print(f"maxpool fwd {fwd * 1e3:.1f} us ({gb_f / fwd * 1e3:.0f} GB/s), "
      f"bwd {bwd * 1e3:.1f} us ({gb_b / bwd * 1e3:.0f} GB/s)")
