"""In-step kernel timing and roofline bookkeeping for bench.py.

Every kernel of the product path is launched by one ``torch.ops.memsave`` op
(paper_2404_12406_b200/_ops.py).  ``trace_step`` swaps the op namespace for a
recorder for ONE extra step after the timed region: each op call is bracketed
by CUDA events on the current stream (the stream the op launches on), and the
GPU is held by a sleep kernel while the host enqueues the step, so every
bracket measures exactly that op's kernels back to back with the rest of the
step (same L2 state, same neighbours) and no host gap.

Algorithmic work per call: GEMM-shaped ops count 2·M·N·K
flops (implicit GEMM for convs: M = N·OH·OW, N = K_out, K = C·R·S) and the
bytes of one read of every operand and one write of every output; bandwidth
ops count the bytes they must move (16-bit elements, 1 bit per ReLU mask
element, 1 byte per pool index).  The bound of a call is the larger of
flops / tensor peak and bytes / HBM peak.
"""

from __future__ import annotations

import math
from collections import OrderedDict

import torch
import torch.utils._python_dispatch  # noqa: F401  (TorchDispatchMode)

from paper_2404_12406_b200 import _ops as OPS


def _numel(shape):
    return int(math.prod(shape))


def _conv_work(xs, ws, stride, pad, es):
    n, c, h, w = xs
    k, _, r, s = ws
    oh = (h + 2 * pad[0] - r) // stride[0] + 1
    ow = (w + 2 * pad[1] - s) // stride[1] + 1
    flops = 2.0 * n * oh * ow * k * c * r * s
    ys = (n, k, oh, ow)
    byts = es * (_numel(xs) + _numel(ws) + _numel(ys))
    return flops, byts, ys


# ops whose backward is a C++ autograd node: their Python-level call is the
# forward, recorded under the forward kernel op's name
_AUTOGRAD_FWD = {"linear": "linear_fwd", "linear_gelu": "linear_gelu_fwd",
                 "linear_dropout_add": "linear_dropout_add_fwd"}


def work_of(name, args):
    """(flops, bytes, geometry) of one op call, from its arguments."""
    def es_of(t):
        return t.element_size()

    a = args
    if name == "linear_bwd":  # (x_shape, w_shape, dtype size, need_dx, need_dw)
        xs, ws_, es, ndx, ndw = a
        N, K = ws_
        M = int(math.prod(xs)) // K
        n = int(ndx) + int(ndw)
        return 2.0 * M * N * K * n, es * n * (M * K + N * K + M * N), dict(M=M, N=N, K=K)
    name = _AUTOGRAD_FWD.get(name, name)
    if name in ("linear_gelu_fwd", "linear_dropout_add_fwd"):
        x, w = a[0], a[1]
        N, K = w.shape
        M = x.numel() // K
        es = es_of(x)
        # + the GELU's second output / the residual read
        return 2.0 * M * N * K, es * (M * K + N * K + 2 * M * N), dict(M=M, N=N, K=K)
    if name in ("linear_fwd", "linear_dx", "linear_dw"):
        if name == "linear_fwd":
            x, w = a[0], a[1]
            N, K = w.shape
            M = x.numel() // K
        elif name == "linear_dx":
            g, w = a[0], a[1]
            N, K = w.shape
            M = g.numel() // N
        else:
            x, g = a[0], a[1]
            K, N = x.shape[-1], g.shape[-1]
            M = g.numel() // N
        es = es_of(a[0])
        return 2.0 * M * N * K, es * (M * K + N * K + M * N), dict(M=M, N=N, K=K)
    if name in ("conv2d_fwd", "conv2d_bn_fwd", "conv2d_dx", "conv2d_bn_dx", "conv2d_dw",
                "conv_transpose2d_fwd"):
        t0 = a[0]
        es = es_of(t0)
        if name == "conv2d_fwd":
            xs, ws, st, pd = tuple(t0.shape), tuple(a[1].shape), a[3], a[4]
        elif name == "conv2d_bn_fwd":
            xs, ws, st, pd = tuple(t0.shape), tuple(a[1].shape), a[11], a[12]
        elif name == "conv2d_dx":
            xs, ws, st, pd = tuple(a[2]), tuple(a[1].shape), a[3], a[4]
        elif name == "conv2d_bn_dx":
            xs, ws, st, pd = tuple(a[11]), tuple(a[1].shape), a[12], a[13]
        elif name == "conv2d_dw":
            xs, ws, st, pd = tuple(t0.shape), tuple(a[2]), a[3], a[4]
        else:  # conv_transpose2d_fwd: the conv whose input-VJP it is
            xs, ws, st, pd = tuple(a[3]), tuple(a[1].shape), a[4], a[5]
        flops, byts, ys = _conv_work(xs, ws, st, pd, es)
        if name == "conv2d_bn_fwd":
            if a[8] is not None:
                byts += es * _numel(ys)           # residual read
            if a[9] and a[10]:
                byts += _numel(ys) / 8.0          # ReLU keep bits
        if name == "conv2d_bn_dx":
            if a[5] is not None:
                byts += es * _numel(xs)           # addend read
            if a[6] is not None:
                byts += _numel(xs) / 8.0          # keep bits
        return flops, byts, dict(x=list(xs), w=list(ws), stride=list(st), pad=list(pd))
    t0 = a[0]
    n = t0.numel()
    es = es_of(t0)
    if name == "bn_eval_fwd":
        return 2.0 * n, 2.0 * es * n, dict(shape=list(t0.shape))
    if name == "bn_eval_bwd":
        need_dx, need_dw = a[7], a[8]
        return 3.0 * n, es * n * (1 + need_dx + need_dw), dict(shape=list(t0.shape))
    if name == "bn_relu_fwd":
        return 3.0 * n, es * n * (2 + (a[1] is not None)) + (n / 8.0 if a[7] else 0), \
            dict(shape=list(t0.shape))
    if name == "bn_add_relu_bwd":
        need_dx, need_dr, need_dw = a[7], a[8], a[9]
        return 3.0 * n, es * n * (1 + need_dx + need_dr + need_dw) + n / 8.0, \
            dict(shape=list(t0.shape))
    if name in ("bn_relu_bwd", "relu_bwd"):
        return float(n), 2.0 * es * n + n / 8.0, dict(shape=list(t0.shape))
    if name in ("relu_fwd", "relu_fwd_"):
        return float(n), 2.0 * es * n + (n / 8.0 if a[1] else 0), dict(shape=list(t0.shape))
    if name == "add_relu_fwd":
        return float(n), 3.0 * es * n + (n / 8.0 if a[2] else 0), dict(shape=list(t0.shape))
    if name == "maxpool2d_fwd":
        k, s, p = a[1], a[2], a[3]
        nb, c, h, w = t0.shape
        oh = (h + 2 * p[0] - k[0]) // s[0] + 1
        ow = (w + 2 * p[1] - k[1]) // s[1] + 1
        ny = nb * c * oh * ow
        return float(ny * k[0] * k[1]), es * (n + ny) + (ny if a[5] else 0), \
            dict(shape=list(t0.shape))
    if name in ("maxpool2d_bwd", "maxpool2d_relu_bwd"):
        xs = a[2] if name == "maxpool2d_bwd" else a[7]
        nx = _numel(xs)
        extra = nx / 8.0 if name == "maxpool2d_relu_bwd" else 0
        return float(nx), es * (n + nx) + n + extra, dict(x=list(xs))
    if name == "gelu_fwd":
        return 20.0 * n, 2.0 * es * n, dict(shape=list(t0.shape))
    if name == "gelu_bwd":
        return 30.0 * n, 3.0 * es * n, dict(shape=list(t0.shape))
    if name in ("dropout_fwd", "dropout_fwd_", "dropout_bwd"):
        return float(n), 2.0 * es * n, dict(shape=list(t0.shape))
    if name == "layernorm_fwd":
        return 8.0 * n, 2.0 * es * n, dict(shape=list(t0.shape))
    if name == "layernorm_bwd":
        return 10.0 * n, es * n * (2 + bool(a[6])), dict(shape=list(t0.shape))
    if name in ("bias_grad", "conv2d_db"):
        return float(n), es * n, dict(shape=list(t0.shape))
    return 0.0, 0.0, {}


class _Recorder:
    """Brackets every torch.ops.memsave call with CUDA events.  memsave::linear
    (and the fused linear_gelu / linear_dropout_add) run their backward in C++
    (csrc/torch_ops.cpp), invisible to this wrapper: the forward call is timed
    under the forward kernel op's name, and hooks on the output's grad_fn time
    the kernel ops its backward node dispatches."""

    def __init__(self, real):
        self._real = real
        self.calls = []

    def __getattr__(self, name):
        fn = getattr(self._real, name)

        def wrapped(*args):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            out = fn(*args)
            e.record()
            flops, byts, geom = work_of(name, args)
            self.calls.append((_AUTOGRAD_FWD.get(name, name), s, e, flops, byts, geom))
            if name in _AUTOGRAD_FWD and out.grad_fn is not None:
                self._hook_backward(out, args)
            return out
        return wrapped

    def _hook_backward(self, out, args):
        # a dispatch mode active only while this backward node runs (on the
        # autograd thread) times each kernel op the C++ backward calls
        node = out.grad_fn
        state = {}

        def pre(grad_outputs):
            state["mode"] = _DispatchRecorder(self)
            state["mode"].__enter__()

        def post(grad_inputs, grad_outputs):
            state.pop("mode").__exit__(None, None, None)

        node.register_prehook(pre)
        node.register_hook(post)


class _DispatchRecorder(torch.utils._python_dispatch.TorchDispatchMode):
    """Times the memsave kernel ops dispatched from C++ (memsave::linear's
    backward: bias_grad, linear_dx, linear_dw)."""

    def __init__(self, rec):
        super().__init__()
        self.rec = rec

    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        if func.namespace != "memsave":
            return func(*args, **kwargs)
        name = func._opname
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        out = func(*args, **kwargs)
        e.record()
        flops, byts, geom = work_of(name, args)
        self.rec.calls.append((name, s, e, flops, byts, geom))
        return out


def trace_step(step, dev, sleep_s: float = 0.3):
    """Run step() once with every memsave op bracketed by CUDA events; returns
    (per-call list, device ms of the whole step)."""
    real = OPS.ops()
    rec = _Recorder(real)
    torch.cuda.synchronize(dev)
    torch.cuda._sleep(int(1.9e9 * sleep_s))  # the host enqueues the whole step meanwhile
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    OPS._OV = rec
    try:
        s0.record()
        step()
        s1.record()
    finally:
        OPS._OV = real
    torch.cuda.synchronize(dev)
    calls = [(n, s.elapsed_time(e), f, b, g) for (n, s, e, f, b, g) in rec.calls]
    return calls, s0.elapsed_time(s1)


def summarise(calls, step_ms, peaks):
    """Group calls by (op, geometry); pick the dominant group (total time) and
    express it against its roofline."""
    groups = OrderedDict()
    for name, ms, flops, byts, geom in calls:
        key = (name, repr(sorted(geom.items())))
        g = groups.setdefault(key, dict(op=name, geom=geom, n=0, ms=0.0, flops=flops, bytes=byts))
        g["n"] += 1
        g["ms"] += ms
    rows = []
    for g in groups.values():
        mean_ms = g["ms"] / g["n"]
        t_tensor = g["flops"] / (peaks["tflops"] * 1e12)
        t_hbm = g["bytes"] / (peaks["gbs"] * 1e9)
        bound = "tensor" if t_tensor >= t_hbm else "hbm"
        if bound == "tensor":
            ach, peak, unit = g["flops"] / (mean_ms * 1e-3) / 1e12, peaks["tflops"], "TFLOP/s"
        else:
            ach, peak, unit = g["bytes"] / (mean_ms * 1e-3) / 1e9, peaks["gbs"], "GB/s"
        rows.append(dict(op=g["op"], geom=g["geom"], launches_per_step=g["n"],
                         ms_per_launch=round(mean_ms, 5), ms_per_step=round(g["ms"], 4),
                         flops=g["flops"], bytes=g["bytes"], bound=bound,
                         achieved=round(ach, 2), peak=peak, unit=unit,
                         frac=round(ach / peak, 4)))
    rows.sort(key=lambda r: -r["ms_per_step"])
    op_ms = sum(r["ms_per_step"] for r in rows)
    return rows, op_ms
