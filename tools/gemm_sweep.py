"""Times bf16 linear_fwd over a list of (M, N, K) (CUDA events, 50 reps): how
the per-tile cost scales with K at BERT's 768-wide output.
python tools/gemm_sweep.py [M,N,K ...]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2404_12406_b200._ops import ops  # noqa: E402

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [
    (32768, 768, 768), (32768, 768, 1536), (32768, 768, 3072), (32768, 1536, 768),
    (32768, 2304, 768), (65536, 768, 768), (16384, 768, 768)]
o = ops()
for M, N, K in shapes:
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / K ** 0.5
    for _ in range(5):
        o.linear_fwd(x, w, None)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        o.linear_fwd(x, w, None)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    print(f"{M:6d} {N:5d} {K:5d}  {us:8.1f} us  {2.0 * M * N * K / us / 1e6:7.1f} TF/s")
