"""CPU port of the benchmark workloads on the reference algorithm — used ONLY
by bench.py's ``cpu_baseline`` leg and by ``bench.py --impl reference``.

``port_model`` takes the workload's own torch model (CPU, float32 -- the dtype
the reference computes in) and swaps every hot-path layer for a port: Conv2d
runs the reference's own kernels (``leantape.kernels`` conv2d_fwd / dx / dw,
installed under baseline/_ref, numpy backend on every host core) or, when that
install is absent, their oracle restatement (oracle/conv.py, numpy_impl.py:12-51);
Linear and BatchNorm2d-eval, which the reference specifies but does not ship
(SPEC.md:241-274), run the oracle restatement (oracle/linear.py, batchnorm.py).
All three keep the reference's selective-save rule (rules.py:133-141).  The
glue between them (ReLU, pooling, attention, LayerNorm, GELU, embedding) stays
torch-CPU.
"""

from __future__ import annotations

import time

import numpy as np

import oracle

F32 = np.float32


def time_cpu(fn, min_seconds: float = 10.0, max_iters: int = 50):
    """Run fn() until min_seconds have elapsed (at least once); returns
    (seconds per call, calls)."""
    fn()  # warm-up (BLAS thread pools, page faults)
    t0 = time.perf_counter()
    n = 0
    while True:
        fn()
        n += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or n >= max_iters:
            return el / n, n


# ---------------------------------------------------------------------------------
# Generic port: the workload's own torch model on the CPU in float32, with every
# layer of the hot path (Conv2d, Linear, BatchNorm2d-eval) computed by the oracle
# restatement of the reference algorithm (numpy_impl.py:12-51 conv, SPEC.md:241-274
# Linear / BN-eval) under the same selective-save rule (rules.py:133-141); the
# glue (ReLU, pooling, attention, LayerNorm, GELU, embedding) stays torch-CPU.
import torch  # noqa: E402
from torch import nn  # noqa: E402


def _np32(t):
    return t.detach().numpy().astype(F32, copy=False)


_REF = None


def reference_kernels():
    """The reference's own conv kernels (``leantape.kernels``, kernels/__init__.py:26-28)
    from the git-ignored install under baseline/_ref (``pip install --target
    baseline/_ref /root/reference``), on its numpy backend (LEANTAPE_JIT=0: np.pad +
    einsum over OpenBLAS, every host core; the numba backend is single-threaded).
    None when the install is absent -- the oracle restatement is used instead."""
    global _REF
    if _REF is None:
        import os
        import sys
        root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "baseline", "_ref")
        try:
            if os.path.isdir(root) and root not in sys.path:
                sys.path.insert(0, root)
            os.environ.setdefault("LEANTAPE_JIT", "0")
            import leantape.kernels as K
            _REF = K
        except Exception:
            _REF = False
    return _REF or None


def _conv_fwd(x, w, stride, pad):
    K = reference_kernels()
    if K is not None:
        return K.conv2d_fwd(np.ascontiguousarray(x), np.ascontiguousarray(w), stride, pad)
    return oracle.conv2d_fwd(x, w, stride, pad, dtype=F32)


def _conv_dx(g, w, stride, pad, h, wd):
    K = reference_kernels()
    if K is not None:
        return K.conv2d_dx(np.ascontiguousarray(g), np.ascontiguousarray(w), stride, pad, h, wd)
    return oracle.conv2d_dx(g, w, stride, pad, h, wd, dtype=F32)


def _conv_dw(x, g, stride, pad, kh, kw):
    K = reference_kernels()
    if K is not None:
        return K.conv2d_dw(np.ascontiguousarray(x), np.ascontiguousarray(g), stride, pad, kh, kw)
    return oracle.conv2d_dw(x, g, stride, pad, kh, kw, dtype=F32)


class _PortConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, stride, pad):
        x_rg, w_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        ctx.save_for_backward(x if w_rg else None, w if x_rg else None)
        ctx.geo = (stride, pad, x.shape)
        ctx.kshape = (w.shape[2], w.shape[3])
        y = _conv_fwd(_np32(x), _np32(w), stride, pad)
        if b is not None:
            y = y + _np32(b)[None, :, None, None]
        return torch.from_numpy(np.ascontiguousarray(y, dtype=F32))

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        stride, pad, xs = ctx.geo
        gn = _np32(g.contiguous())
        dx = dw = db = None
        if ctx.needs_input_grad[0]:
            dx = torch.from_numpy(_conv_dx(gn, _np32(w), stride, pad, xs[2], xs[3]).astype(F32))
        if ctx.needs_input_grad[1]:
            dw = torch.from_numpy(_conv_dw(_np32(x), gn, stride, pad, *ctx.kshape).astype(F32))
        if ctx.needs_input_grad[2]:
            db = torch.from_numpy(gn.sum(axis=(0, 2, 3)).astype(F32))
        return dx, dw, db, None, None


class _PortConv(nn.Module):
    def __init__(self, conv):
        super().__init__()
        self.conv = conv

    def forward(self, x):
        c = self.conv
        return _PortConvFn.apply(x.contiguous(), c.weight, c.bias, c.stride[0], c.padding[0])


class _PortLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b):
        x_rg, w_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        ctx.save_for_backward(x if w_rg else None, w if x_rg else None)
        y = oracle.linear_fwd(_np32(x), _np32(w), None if b is None else _np32(b), dtype=F32)
        return torch.from_numpy(np.ascontiguousarray(y, dtype=F32))

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        gn = _np32(g.contiguous())
        dx = dw = db = None
        if ctx.needs_input_grad[0]:
            dx = torch.from_numpy(oracle.linear_dx(gn, _np32(w), dtype=F32))
        if ctx.needs_input_grad[1]:
            dw = torch.from_numpy(oracle.linear_dw(_np32(x), gn, dtype=F32))
        if ctx.needs_input_grad[2]:
            db = torch.from_numpy(oracle.linear_db(gn, dtype=F32))
        return dx, dw, db


class _PortLinear(nn.Module):
    def __init__(self, lin):
        super().__init__()
        self.lin = lin

    def forward(self, x):
        return _PortLinearFn.apply(x.contiguous(), self.lin.weight, self.lin.bias)


class _PortBNFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, mean, var, eps):
        x_rg, w_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        ctx.save_for_backward(x if w_rg else None, w if x_rg else None)
        ctx.st = (mean, var, eps)
        y = oracle.bn_eval_fwd(_np32(x), _np32(mean), _np32(var), _np32(w), _np32(b), eps)
        return torch.from_numpy(y.astype(F32))

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        mean, var, eps = ctx.st
        gn = _np32(g.contiguous())
        dx = dw = db = None
        if ctx.needs_input_grad[0]:
            dx = torch.from_numpy(oracle.bn_eval_dx(gn, _np32(var), _np32(w), eps).astype(F32))
        if ctx.needs_input_grad[1]:
            dw = torch.from_numpy(oracle.bn_eval_dw(gn, _np32(x), _np32(mean), _np32(var),
                                                    eps).astype(F32))
        if ctx.needs_input_grad[2]:
            db = torch.from_numpy(oracle.bn_eval_db(gn).astype(F32))
        return dx, dw, db, None, None, None


class _PortBN(nn.Module):
    def __init__(self, bn):
        super().__init__()
        self.bn = bn

    def forward(self, x):
        if self.bn.training:
            return self.bn(x)
        b = self.bn
        return _PortBNFn.apply(x.contiguous(), b.weight, b.bias, b.running_mean,
                               b.running_var, b.eps)


def port_model(model: nn.Module) -> nn.Module:
    """Swap Conv2d / Linear / BatchNorm2d (in place) for their oracle ports."""
    for name, child in list(model.named_children()):
        if type(child) is nn.Conv2d and child.groups == 1 and child.dilation == (1, 1) \
                and not isinstance(child.padding, str):
            setattr(model, name, _PortConv(child))
        elif type(child) is nn.Linear:
            setattr(model, name, _PortLinear(child))
        elif type(child) is nn.BatchNorm2d:
            setattr(model, name, _PortBN(child))
        else:
            port_model(child)
    return model


def _isa() -> str:
    try:
        flags = open("/proc/cpuinfo").read().split("flags", 2)[1].split("\n", 1)[0]
        have = [f for f in ("avx2", "avx512f", "avx512_bf16", "amx_bf16", "amx_tile")
                if f" {f}" in flags]
        return "x86_64 " + "+".join(have)
    except Exception:
        import platform
        return platform.machine()


def cpu_workload(config: str):
    """(step, record): ``step()`` runs one bounded sample of ``config`` through the
    CPU port on all host threads and returns the seconds it implies per sample
    of the full workload; ``record`` describes the sample (cpu_baseline keys)."""
    import os

    from benchkit import models as BM
    torch.manual_seed(0)
    torch.set_num_threads(os.cpu_count() or 1)
    K = reference_kernels()
    conv_src = ("reference leantape.kernels (numpy backend)" if K is not None
                else "oracle restatement of numpy_impl.py:12-51")
    rec = {"unit": "samples/s", "cores": torch.get_num_threads(), "isa": _isa(), "dtype": "f32"}
    if config == "llama":
        return _llama_workload(rec)
    batch = 1
    wl = BM.WORKLOADS[config](batch=batch, dtype=torch.float32, device="cpu")
    model = port_model(wl.model)
    ins = list(wl.make_batch(batch, torch.device("cpu")))

    def step():
        t0 = time.perf_counter()
        if wl.input_requires_grad:
            ins[0].requires_grad_(True)
            ins[0].grad = None
        for p in model.parameters():
            p.grad = None
        wl.loss_fn(model, *ins).backward()
        return (time.perf_counter() - t0) / batch

    uses_conv = config in ("fig1", "resnet18", "resnet101", "vgg16")
    rec.update(kind="reference" if (uses_conv and K is not None) else "port",
               sample=(f"fwd+bwd of {batch} sample of the {config} workload (same model, "
                       f"trainable set and loss) in float32; conv: {conv_src}; Linear / "
                       f"BN-eval: oracle restatement of SPEC.md:241-274 (no reference code); "
                       f"glue ops torch-CPU"))
    return step, rec


def cpu_sample(config: str, min_seconds: float = 10.0) -> dict:
    """The cpu_baseline record: the CPU port timed for about ``min_seconds``."""
    step, rec = cpu_workload(config)
    step()  # warm-up (BLAS thread pools, page faults)
    t0 = time.perf_counter()
    per = []
    while not per or (time.perf_counter() - t0 < min_seconds and len(per) < 50):
        per.append(step())
    sec = sum(per) / len(per)
    rec.update(value=round(1.0 / sec, 6), seconds_per_sample=round(sec, 4),
               sample=f"{len(per)} x " + rec["sample"])
    return rec


def _llama_workload(rec: dict):
    """Llama-3-8B is too large for a whole-model CPU step: one sample times one
    decoder layer (frozen: forward only; trainable: forward + backward with dW and
    dX) and the head (final norm + lm_head + loss, forward + backward) on 1
    sequence of 512 tokens; per 2048-token sequence = 4 x (28 frozen + 4
    trainable layers + head)."""
    from benchkit import models as BM
    wl = BM.llama3_8b_last4(batch=1, seq=512, dtype=torch.float32, device="cpu", layers=1)
    model = port_model(wl.model)
    layer = model.model.layers[0]
    h = torch.randn(1, 512, 4096)
    pos = torch.arange(512)[None]
    pe = model.model.rotary_emb(h, pos)
    ids = torch.randint(0, 128256, (1, 512))

    def frozen_layer():
        with torch.no_grad():
            layer(h, position_embeddings=pe, position_ids=pos)

    def trainable_layer():
        for p in layer.parameters():
            p.grad = None
        hh = h.clone().requires_grad_(True)
        out = layer(hh, position_embeddings=pe, position_ids=pos)
        out = out[0] if isinstance(out, tuple) else out
        out.float().sum().backward()

    def head():
        hh = h.clone().requires_grad_(True)
        logits = model.lm_head(model.model.norm(hh))
        torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), ids.view(-1)) \
            .backward()

    def timed(fn):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    def step():
        tf, tt, th = timed(frozen_layer), timed(trainable_layer), timed(head)
        return 4.0 * (28 * tf + 4 * tt + th)

    rec.update(kind="port",
               sample=("1 x 512-token sequence through one decoder layer forward (frozen), one "
                       "forward+backward (trainable) and the head; per 2048-token sequence = "
                       "4 x (28 frozen + 4 trainable + head); Linear: oracle restatement of "
                       "SPEC.md:241-249, glue torch-CPU"))
    return step, rec
