"""Dropout / LayerNorm kernels vs torch on the BERT shapes (32768 x 768 bf16)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from benchkit.kernels import time_launches  # noqa: E402
from paper_2404_12406_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
rows, d = 32768, 768
x = torch.randn(rows, d, device=dev, dtype=torch.bfloat16)
y = torch.empty_like(x)
n = x.numel()
ref = time_launches(lambda: torch.nn.functional.dropout(x, 0.1, True), 20, dev)
for gen, name in ((0, "philox4x32"), (1, "reference philox4x64")):
    ours = time_launches(lambda: L.ms_dropout_fwd(n, 1, P(x), P(y), 123, 1000000, 0.1, gen, None,
                                                  st), 20, dev)
    print(f"dropout fwd {n} bf16 [{name}]: ours {ours * 1e3:.1f} us "
          f"({4 * n / ours / 1e6:.0f} GB/s) | torch {ref * 1e3:.1f} us")
w = torch.randn(d, device=dev, dtype=torch.bfloat16)
b = torch.randn(d, device=dev, dtype=torch.bfloat16)
mean = torch.empty(rows, device=dev)
rstd = torch.empty(rows, device=dev)
ours = time_launches(lambda: L.ms_layernorm_fwd(rows, d, 1, P(x), P(w), P(b), 1e-5, P(y), P(mean),
                                                P(rstd), st), 20, dev)
ref = time_launches(lambda: torch.nn.functional.layer_norm(x, (d,), w, b), 20, dev)
print(f"layernorm fwd: ours {ours * 1e3:.1f} us ({4 * n / ours / 1e6:.0f} GB/s) | "
      f"torch {ref * 1e3:.1f} us")
g = torch.randn_like(x)
dx = torch.empty_like(x)
ours = time_launches(lambda: L.ms_layernorm_bwd(rows, d, 1, P(g), P(x), P(mean), P(rstd), P(w),
                                                P(dx), None, None, None, 0, st), 20, dev)
xr = x.clone().requires_grad_(True)
yr = torch.nn.functional.layer_norm(xr, (d,), w, b)
ref = time_launches(lambda: torch.autograd.grad(yr, xr, g, retain_graph=True), 20, dev)
print(f"layernorm bwd (dx): ours {ours * 1e3:.1f} us ({6 * n / ours / 1e6:.0f} GB/s) | "
      f"torch {ref * 1e3:.1f} us")
