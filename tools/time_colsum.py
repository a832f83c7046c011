"""Device time of the bias-gradient column sum (memsave::bias_grad) at BERT's
32768 x 768 and a few other shapes, CUDA events over 50 calls."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2404_12406_b200._ops import ops  # noqa: E402

O = ops()
for rows, cols in ((32768, 768), (32768, 3072), (4096, 4096), (128 * 196, 256)):
    g = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        O.bias_grad(g, cols)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        O.bias_grad(g, cols)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    print(f"colsum {rows}x{cols}: {us:6.1f} us  {rows * cols * 2 / us / 1e3:6.0f} GB/s")
