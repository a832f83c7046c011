"""Run one linear pass a few times (for ncu captures):
python tools/one_linear.py M N K [fwd|fwdb|dx|dw] [reps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_12406_b200 import _lib  # noqa: E402

M, N, K = map(int, sys.argv[1:4])
which = sys.argv[4] if len(sys.argv) > 4 else "fwdb"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
dev = torch.device("cuda", 0)
L = _lib.lib()
st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
x = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
w = torch.randn(N, K, device=dev, dtype=torch.bfloat16) * 0.02
b = torch.randn(N, device=dev, dtype=torch.bfloat16)
y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
dy = torch.randn(M, N, device=dev, dtype=torch.bfloat16)
dx = torch.empty(M, K, device=dev, dtype=torch.bfloat16)
dw = torch.empty(N, K, device=dev, dtype=torch.bfloat16)
nbw = max(L.ms_linear_workspace(M, N, K, 1, 2), 1)
ws = torch.empty(nbw, dtype=torch.uint8, device=dev)
fn = {
    "fwd": lambda: L.ms_linear_fwd(M, N, K, 1, P(x), P(w), None, P(y), None, 0, st),
    "fwdb": lambda: L.ms_linear_fwd(M, N, K, 1, P(x), P(w), P(b), P(y), None, 0, st),
    "dx": lambda: L.ms_linear_dx(M, N, K, 1, P(dy), P(w), P(dx), None, 0, st),
    "dw": lambda: L.ms_linear_dw(M, N, K, 1, P(x), P(dy), P(dw), P(ws), nbw, st),
}[which]
for _ in range(reps):
    assert fn() == 0
torch.cuda.synchronize()
print("ok")
