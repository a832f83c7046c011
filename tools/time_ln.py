"""LayerNorm fwd / input-VJP at BERT size (32768 x 768 bf16), device time per
call from a captured CUDA graph, against the bytes each must move."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2404_12406_b200._ops import ops  # noqa: E402

dev = torch.device("cuda", 0)
O = ops()
x = torch.randn(32768, 768, device=dev, dtype=torch.bfloat16)
g = torch.randn_like(x)
w = torch.randn(768, device=dev, dtype=torch.bfloat16)
b = torch.randn(768, device=dev, dtype=torch.bfloat16)
_, mean, rstd = O.layernorm_fwd(x, w, b, 1e-12, 768, True)


def timed(fn, reps=20):
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


nb = x.numel() * 2
us = timed(lambda: O.layernorm_fwd(x, w, b, 1e-12, 768, True))
print(f"ln fwd {us:.1f} us  {2 * nb / us / 1e3:.0f} GB/s")
us = timed(lambda: O.layernorm_bwd(g, x, mean, rstd, w, 768, True, False, False))
print(f"ln bwd dx {us:.1f} us  {3 * nb / us / 1e3:.0f} GB/s")
