"""Time the Fig.1 conv kernels (fwd, and fwd+dX+dW via backward) at (32,8,256,256)
fp32: back-to-back launches between two events (inputs > L2)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2404_12406_b200 import functional as MF  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.randn((32, 8, 256, 256), device=dev)
w = torch.randn((8, 8, 3, 3), device=dev) / 24
g = torch.randn((32, 8, 256, 256), device=dev)


def timed(fn, reps=20):
    """device time per call: `reps` calls captured in one CUDA graph (no host
    launch overhead in the measurement)"""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    gr.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


us = timed(lambda: MF.conv2d(x, w, None, 1, 1))
print(f"fwd {us:.1f} us  {134.2e6 / us / 1e3:.0f} GB/s", flush=True)
from paper_2404_12406_b200._ops import ops  # noqa: E402

O = ops()
geo = ([1, 1], [1, 1], 0, 0)  # NCHW, OIHW
us = timed(lambda: O.conv2d_fwd(x, w, None, *geo))
print(f"fwd (op) {us:.1f} us  {134.2e6 / us / 1e3:.0f} GB/s", flush=True)
us = timed(lambda: O.conv2d_dx(g, w, list(x.shape), *geo))
print(f"dx (op) {us:.1f} us  {134.2e6 / us / 1e3:.0f} GB/s", flush=True)
us = timed(lambda: O.conv2d_dw(x, g, list(w.shape), *geo))
print(f"dw (op) {us:.1f} us  {134.2e6 / us / 1e3:.0f} GB/s", flush=True)
