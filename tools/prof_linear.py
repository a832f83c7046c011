"""Linear (tcgen05 GEMM) vs torch/cuBLAS on the BERT / Llama shapes:
python tools/prof_linear.py [names...]  (M, N, K) = rows, out_features, in_features"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from benchkit.kernels import time_launches  # noqa: E402
from paper_2404_12406_b200 import _lib  # noqa: E402

SHAPES = {
    "bert_qkv": (32768, 768, 768), "bert_ffn1": (32768, 3072, 768),
    "bert_ffn2": (32768, 768, 3072),
    "llama_q": (4096, 4096, 4096), "llama_kv": (4096, 1024, 4096),
    "llama_up": (4096, 14336, 4096), "llama_down": (4096, 4096, 14336),
    "llama_head": (4096, 128256, 4096), "sq8k": (8192, 8192, 8192),
}
dev = torch.device("cuda", 0)
L = _lib.lib()
st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
for name in (sys.argv[1:] or list(SHAPES)):
    M, N, K = SHAPES[name]
    x = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    w = torch.randn(N, K, device=dev, dtype=torch.bfloat16) * 0.02
    y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    b = torch.randn(N, device=dev, dtype=torch.bfloat16)
    dy = torch.randn(M, N, device=dev, dtype=torch.bfloat16)
    dx = torch.empty(M, K, device=dev, dtype=torch.bfloat16)
    dw = torch.empty(N, K, device=dev, dtype=torch.bfloat16)
    out = []
    nb0 = max(L.ms_linear_workspace(M, N, K, 1, 0), 1)
    nb1 = max(L.ms_linear_workspace(M, N, K, 1, 1), 1)
    ws0 = torch.empty(nb0, dtype=torch.uint8, device=dev)
    ws1 = torch.empty(nb1, dtype=torch.uint8, device=dev)
    for ps, fn_ours, fn_ref in (
        ("fwd", lambda: L.ms_linear_fwd(M, N, K, 1, P(x), P(w), None, P(y), P(ws0), nb0, st),
         lambda: torch.matmul(x, w.t(), out=y)),
        ("fwd+bias", lambda: L.ms_linear_fwd(M, N, K, 1, P(x), P(w), P(b), P(y), P(ws0), nb0, st),
         lambda: torch.addmm(b, x, w.t(), out=y)),
        ("dx", lambda: L.ms_linear_dx(M, N, K, 1, P(dy), P(w), P(dx), P(ws1), nb1, st),
         lambda: torch.matmul(dy, w, out=dx)),
    ):
        ms = time_launches(fn_ours, 10, dev)
        ref = time_launches(fn_ref, 10, dev)
        fl = 2.0 * M * N * K
        out.append(f"{ps}: ours {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s | cublas {ref:.3f} ms "
                   f"{fl / ref / 1e9:.0f} TF/s")
    nbw = max(L.ms_linear_workspace(M, N, K, 1, 2), 1)
    ws = torch.empty(nbw, dtype=torch.uint8, device=dev)
    ms = time_launches(lambda: L.ms_linear_dw(M, N, K, 1, P(x), P(dy), P(dw), P(ws), nbw, st),
                       10, dev)
    ref = time_launches(lambda: torch.matmul(dy.t(), x, out=dw), 10, dev)
    fl = 2.0 * M * N * K
    out.append(f"dw: ours {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s | cublas {ref:.3f} ms "
               f"{fl / ref / 1e9:.0f} TF/s")
    print(name, (M, N, K), " || ".join(out), flush=True)
