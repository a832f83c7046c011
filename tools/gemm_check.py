"""Correctness sweep of the tcgen05 linear kernels against torch (fp32 accumulate
reference) over shapes / tile configs; each shape in its own subprocess so a
trapped kernel does not take the others down.
python tools/gemm_check.py [M N K ...]"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [(256, 64, 64), (256, 128, 128), (512, 192, 256), (384, 768, 768), (2048, 768, 768),
          (32768, 768, 768), (4096, 4096, 4096)]


def one(M, N, K):
    import torch
    from paper_2404_12406_b200 import _lib
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(M, K, device=dev, dtype=torch.bfloat16, generator=g)
    w = torch.randn(N, K, device=dev, dtype=torch.bfloat16, generator=g)
    dy = torch.randn(M, N, device=dev, dtype=torch.bfloat16, generator=g)
    y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    dx = torch.empty(M, K, device=dev, dtype=torch.bfloat16)
    dw = torch.empty(N, K, device=dev, dtype=torch.bfloat16)
    nb = [max(L.ms_linear_workspace(M, N, K, 1, i), 1) for i in range(3)]
    ws = [torch.empty(n, dtype=torch.uint8, device=dev) for n in nb]
    out = []
    for name, fn, got, ref in (
        ("fwd", lambda: L.ms_linear_fwd(M, N, K, 1, P(x), P(w), None, P(y), P(ws[0]), nb[0], st), y,
         lambda: x.float() @ w.float().t()),
        ("dx", lambda: L.ms_linear_dx(M, N, K, 1, P(dy), P(w), P(dx), P(ws[1]), nb[1], st), dx,
         lambda: dy.float() @ w.float()),
        ("dw", lambda: L.ms_linear_dw(M, N, K, 1, P(x), P(dy), P(dw), P(ws[2]), nb[2], st), dw,
         lambda: dy.float().t() @ x.float()),
    ):
        rc = fn()
        torch.cuda.synchronize()
        r = ref()
        err = ((got.float() - r).norm() / r.norm()).item()
        print(f"{M}x{N}x{K} {name} rc={rc} rel={err:.2e}{' BAD' if err > 5e-3 or rc else ''}",
              flush=True)


if __name__ == "__main__":
    if len(sys.argv) == 5 and sys.argv[1] == "--one":
        one(*map(int, sys.argv[2:]))
        sys.exit(0)
    args = list(map(int, sys.argv[1:]))
    shapes = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)] or SHAPES
    for s in shapes:
        try:
            r = subprocess.run([sys.executable, __file__, "--one", *map(str, s)], timeout=180,
                               capture_output=True, text=True)
            lines = (r.stdout + r.stderr).strip().splitlines()
            lines = [ln for ln in lines if "watchdog" not in ln]
            print(" | ".join(lines[-3:]) if r.returncode == 0 else
                  f"{s}: FAILED rc={r.returncode}: " + " | ".join(lines[-4:]), flush=True)
        except subprocess.TimeoutExpired as e:
            print(f"{s}: TIMEOUT " + str(e.stdout), flush=True)
