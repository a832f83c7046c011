"""float32 Linear: the tcgen05 3xTF32 path vs the CUDA-core path (MS_FP32_LINEAR=simt)
and vs cuBLAS fp32 (TF32 off), device time per call from a captured CUDA graph."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2404_12406_b200._ops import ops  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
O = ops()


def timed(fn, reps=10):
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
    return s.elapsed_time(e) / reps


for (M, N, K) in [(4096, 4096, 4096), (32768, 768, 768), (8192, 3072, 768), (512, 1000, 2048)]:
    x = torch.randn(M, K, device=dev)
    w = torch.randn(N, K, device=dev) / K ** 0.5
    ours = timed(lambda: O.linear_fwd(x, w, None))
    ref = timed(lambda: torch.matmul(x, w.t()))
    fl = 2.0 * M * N * K
    print(f"({M},{N},{K}) fwd ours {ours:.3f} ms {fl / ours / 1e9:.0f} TF/s | cuBLAS fp32 {ref:.3f} ms "
          f"{fl / ref / 1e9:.0f} TF/s", flush=True)
