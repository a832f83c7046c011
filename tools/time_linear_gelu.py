"""Times the Linear -> GELU pieces at the BERT FFN shape (CUDA events, graph-free):
linear_fwd, the fused linear_gelu_fwd, and the elementwise gelu fwd / bwd.
MS_GEMM_DBG=4 / 8 isolate the epilogue GELU's arithmetic / second store."""
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


M, N, K = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 3072, 768))]
x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / K ** 0.5
b = torch.randn(N, device="cuda", dtype=torch.bfloat16)
ops = torch.ops.memsave
pre = ops.linear_fwd(x, w, b)
g = torch.randn_like(pre)
print(f"shape {M}x{N}x{K}")
print(f"linear_fwd        {t(lambda: ops.linear_fwd(x, w, b)):8.1f} us")
print(f"linear_gelu_fwd   {t(lambda: ops.linear_gelu_fwd(x, w, b)):8.1f} us")
print(f"gelu_fwd          {t(lambda: ops.gelu_fwd(pre)):8.1f} us")
print(f"gelu_bwd          {t(lambda: ops.gelu_bwd(g, pre)):8.1f} us")
print(f"torch gelu        {t(lambda: torch.nn.functional.gelu(pre)):8.1f} us")
print(f"torch gelu_bwd    {t(lambda: torch.ops.aten.gelu_backward(g, pre)):8.1f} us")
