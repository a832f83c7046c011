"""Times the fused Linear -> dropout -> + residual against its parts at BERT's
output-projection shapes (CUDA events): linear_fwd, the fused op at p = 0.1
and p = 0 (residual only), dropout_fwd and torch's add."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2404_12406_b200 import _ops as _O  # noqa: E402

_O._load()


def t(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3


ops = torch.ops.memsave
for M, N, K in ((32768, 768, 768), (32768, 768, 3072)):
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / K ** 0.5
    b = torch.randn(N, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
    y = ops.linear_fwd(x, w, b)
    print(f"shape {M}x{N}x{K}")
    print(f"  linear_fwd              {t(lambda: ops.linear_fwd(x, w, b)):8.1f} us")
    print(f"  fused p=0.1             {t(lambda: ops.linear_dropout_add_fwd(x, w, b, r, 0.1, 5, 1000000, 0)):8.1f} us")
    print(f"  fused p=0 (resid only)  {t(lambda: ops.linear_dropout_add_fwd(x, w, b, r, 0.0, 5, 1000000, 0)):8.1f} us")
    print(f"  dropout_fwd             {t(lambda: ops.dropout_fwd(y, 0.1, 5, 1000000, 0)):8.1f} us")
    print(f"  torch add               {t(lambda: y + r):8.1f} us")
