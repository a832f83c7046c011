"""Per-launch kernel timing through the C ABI (CUDA events on the launching
stream, L2 flushed before every launch) and the roofline bookkeeping bench.py
reports: algorithmic FLOPs / bytes per launch, bound, achieved, fraction."""

from __future__ import annotations

import ctypes

import torch

from paper_2404_12406_b200 import _lib


def _flush_buffer(dev):
    return torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2


def time_launches(fn, reps: int, dev, flush: bool = True) -> float:
    """Mean device time (ms) of fn() over reps launches, each preceded by an
    L2 flush that is outside the timed window."""
    buf = _flush_buffer(dev) if flush else None
    fn()
    torch.cuda.synchronize(dev)
    evs = []
    for _ in range(reps):
        if buf is not None:
            buf.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize(dev)
    return sum(s.elapsed_time(e) for s, e in evs) / reps


def conv_roofline(n, c, h, w, k, r, stride, pad, dev, peaks, reps=10,
                  passes=("fwd", "dx"), dtype=torch.bfloat16):
    """Time ms_conv2d_fwd / ms_conv2d_dx for one geometry (NHWC bf16)."""
    L = _lib.lib()
    oh = (h + 2 * pad - r) // stride + 1
    ow = (w + 2 * pad - r) // stride + 1
    cl = torch.channels_last
    x = torch.randn(n, c, h, w, device=dev, dtype=dtype).contiguous(memory_format=cl)
    wt = (torch.randn(k, c, r, r, device=dev, dtype=dtype) * 0.05).contiguous(memory_format=cl)
    y = torch.empty(n, k, oh, ow, device=dev, dtype=dtype, memory_format=cl)
    dy = torch.randn(n, k, oh, ow, device=dev, dtype=dtype).contiguous(memory_format=cl)
    dx = torch.empty_like(x)
    d = _lib.ConvDesc(n, c, h, w, k, r, r, stride, stride, pad, pad, _lib.MS_NHWC, _lib.MS_NHWC,
                      _lib.MS_BF16)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    es = 2
    flops = 2.0 * n * oh * ow * k * c * r * r
    out = []
    for ps in passes:
        if ps == "fwd":
            nb = L.ms_conv2d_workspace(ctypes.byref(d), _lib.MS_CONV_FWD)
            ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)

            def fn():
                _lib.check(L.ms_conv2d_fwd(ctypes.byref(d), ctypes.c_void_p(x.data_ptr()),
                                           ctypes.c_void_p(wt.data_ptr()), None,
                                           ctypes.c_void_p(y.data_ptr()),
                                           ctypes.c_void_p(ws.data_ptr()), nb, st), "fwd")
            byts = es * (n * c * h * w + k * c * r * r + n * k * oh * ow)
        else:
            nb = L.ms_conv2d_workspace(ctypes.byref(d), _lib.MS_CONV_DX)
            ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)

            def fn():
                _lib.check(L.ms_conv2d_dx(ctypes.byref(d), ctypes.c_void_p(dy.data_ptr()),
                                          ctypes.c_void_p(wt.data_ptr()),
                                          ctypes.c_void_p(dx.data_ptr()),
                                          ctypes.c_void_p(ws.data_ptr()), nb, st), "dx")
            byts = es * (n * c * h * w + k * c * r * r + n * k * oh * ow)
        ms = time_launches(fn, reps, dev)
        out.append(roofline_entry(f"conv_{ps}", dict(n=n, c=c, h=h, w=w, k=k, r=r, stride=stride,
                                                      pad=pad), flops, byts, ms, peaks))
    return out


def roofline_entry(kind, geom, flops, byts, ms, peaks):
    t_tensor = flops / (peaks["tflops"] * 1e12)
    t_hbm = byts / (peaks["gbs"] * 1e9)
    bound = "tensor" if t_tensor >= t_hbm else "hbm"
    sec = ms * 1e-3
    if bound == "tensor":
        achieved, peak, unit = flops / sec / 1e12, peaks["tflops"], "TFLOP/s"
    else:
        achieved, peak, unit = byts / sec / 1e9, peaks["gbs"], "GB/s"
    return dict(kind=kind, geom=geom, flops=flops, bytes=byts, ms=ms, bound=bound,
                achieved=achieved, peak=peak, unit=unit, frac=achieved / peak,
                roofline_ms=max(t_tensor, t_hbm) * 1e3)


def bn_roofline(n, c, hw, dev, peaks, reps=10, dtype=torch.bfloat16):
    """Eval-BN forward and input-VJP (NHWC): pure bandwidth kernels."""
    L = _lib.lib()
    x = torch.randn(n, hw, c, device=dev, dtype=dtype)
    y = torch.empty_like(x)
    m = torch.zeros(c, device=dev, dtype=dtype)
    v = torch.ones(c, device=dev, dtype=dtype)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def fwd():
        _lib.check(L.ms_bn_eval_fwd(n, c, hw, _lib.MS_NHWC, _lib.MS_BF16, _lib.MS_BF16, p(x),
                                    p(m), p(v), p(v), p(m), 1e-5, p(y), None, 0, st), "bn fwd")

    def bwd():
        _lib.check(L.ms_bn_eval_bwd(n, c, hw, _lib.MS_NHWC, _lib.MS_BF16, _lib.MS_BF16, p(x), None,
                                    p(m), p(v), p(v), 1e-5, p(y), None, None, None, 0, st),
                   "bn bwd")
    byts = 2.0 * 2 * n * c * hw
    out = []
    for name, fn in (("bn_fwd", fwd), ("bn_dx", bwd)):
        ms = time_launches(fn, reps, dev)
        out.append(roofline_entry(name, dict(n=n, c=c, hw=hw), 2.0 * n * c * hw, byts, ms, peaks))
    return out
