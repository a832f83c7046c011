"""Per-call host cost (µs) of one conv / linear launch at each layer of the
stack, with the GPU held busy so nothing waits on the device:
C ABI (ctypes) -> torch.ops.memsave op -> autograd.Function -> module."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def per_call_us(fn, n=300):
    import torch
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1.9e9 * 0.3))
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return dt


def main():
    import torch

    from paper_2404_12406_b200 import _lib
    from paper_2404_12406_b200 import functional as MF
    from paper_2404_12406_b200._ops import ops
    O = ops()
    L = _lib.lib()
    cl = torch.channels_last
    x = torch.randn(8, 256, 14, 14, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
    w = torch.randn(256, 256, 3, 3, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
    y = torch.empty_like(x)
    d = _lib.ConvDesc(8, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1, 1, 1, 1)
    nb = L.ms_conv2d_workspace(ctypes.byref(d), 0)
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    xp, wp, yp, wsp = x.data_ptr(), w.data_ptr(), y.data_ptr(), ws.data_ptr()
    res = {}
    res["capi conv fwd (ctypes)"] = per_call_us(
        lambda: L.ms_conv2d_fwd(ctypes.byref(d), xp, wp, None, yp, wsp, nb, st))
    res["torch.ops conv2d_fwd"] = per_call_us(
        lambda: O.conv2d_fwd(x, w, None, [1, 1], [1, 1], 1, 1))
    res["MF.conv2d (no grad)"] = per_call_us(lambda: MF.conv2d(x, w, None, 1, 1))
    res["F.conv2d cuDNN"] = per_call_us(lambda: torch.nn.functional.conv2d(x, w, None, 1, 1))
    a = torch.randn(4096, 1024, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(1024, 1024, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(4096, 1024, device="cuda", dtype=torch.bfloat16)
    nb2 = L.ms_linear_workspace(4096, 1024, 1024, 1, 0)
    ws2 = torch.empty(max(nb2, 1), dtype=torch.uint8, device="cuda")
    res["capi linear fwd (ctypes)"] = per_call_us(
        lambda: L.ms_linear_fwd(4096, 1024, 1024, 1, a.data_ptr(), b.data_ptr(), None,
                                c.data_ptr(), ws2.data_ptr(), nb2, st))
    res["torch.ops linear_fwd"] = per_call_us(lambda: O.linear_fwd(a, b, None))
    res["F.linear cuBLAS"] = per_call_us(lambda: torch.nn.functional.linear(a, b))
    res["torch.empty"] = per_call_us(lambda: torch.empty(4096, 1024, device="cuda"))
    res["relu_fwd op"] = per_call_us(lambda: O.relu_fwd(a, True))
    for k, v in res.items():
        print(f"{k:32s} {v:7.2f} us/call")


if __name__ == "__main__":
    main()
