"""Selective-save autograd functions for Linear, Conv2d and BatchNorm2d (eval).

Each function decides at FORWARD time, from ``ctx.needs_input_grad`` (the
requires_grad flags of its input and weight), which tensors to keep
(rules.saved_roles; reference rules.py:133-141), and its backward launches only
the products that were requested (dX, dW, db).  All arithmetic runs in the
sm_100a kernels of ``libmemsave_b200.so`` through its C ABI; there is no CPU
path.  Tensors on the ``meta`` device are accepted and produce shapes only, so
the storage logic can be exercised without a GPU (no arithmetic is done).

Reference parity (the "layers" module of SPEC.md, which the reference package
specifies but does not ship):
  linear        forward_linear
  conv2d        forward_conv2d        SPEC.md:250-258 (kernels/__init__.py:26-28)
  batch_norm    forward_batchnorm2d   SPEC.md:266-274, eval mode; running
                statistics are module state, not saved tensors
"""

from __future__ import annotations

import os

import torch

from . import _lib
from ._ops import ops as _ops
from .rules import MissingSavedValue, saved_roles

_DT = {torch.float32: _lib.MS_F32, torch.bfloat16: _lib.MS_BF16, torch.float16: _lib.MS_F16}


def _dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"memsave_b200: unsupported dtype {t.dtype}; expected float32, "
                        f"bfloat16 or float16") from None


def _opt(t, want: bool):
    """An op output that is empty when the product was not requested -> None."""
    return t if want else None


def _is_meta(*ts) -> bool:
    return any(t is not None and t.device.type == "meta" for t in ts)


def _require_cuda(what: str, *ts) -> None:
    for t in ts:
        if t is not None and t.device.type != "cuda":
            raise RuntimeError(f"memsave_b200.{what}: tensors must be on a CUDA device (got "
                               f"{t.device}); this implementation has no CPU path")


def _need(t, role: str, what: str):
    if t is None:
        raise MissingSavedValue(f"{what}: backward needs '{role}' but the storage rule did not "
                                f"keep it")
    return t


def _is_channels_last(t: torch.Tensor) -> bool:
    return t.dim() == 4 and t.is_contiguous(memory_format=torch.channels_last)


# =============================================================== linear
def linear(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None = None):
    """Differentiability-agnostic ``F.linear``.

    ``torch.ops.memsave.linear`` is a C++ autograd Function (csrc/torch_ops.cpp,
    ``LinearFn``): at forward time it keeps X only if the weight requires a
    gradient and W only if X does (the linear family, rules.py:133-141), and its
    backward launches only the requested products (dX, dW, db).  CPU tensors
    raise (no CPU path); meta tensors take the same storage decisions without
    arithmetic."""
    return _ops().linear(x, weight, bias)


def linear_gelu(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None = None):
    """``gelu(linear(x))`` (erf GELU, ``approximate='none'``) as one node.

    ``torch.ops.memsave.linear_gelu`` (csrc/torch_ops.cpp, ``LinearGeluFn``)
    writes the pre-activation and the GELU output from the same GEMM epilogue
    instead of a second pass over the pre-activation.  The saved set is the
    union of the two layers' rules: X iff W requires a gradient, W iff X does
    (rules.py:133-141), and the pre-activation (the GELU's input, which its VJP
    reads).  Values equal ``gelu(linear(x))`` computed op by op."""
    return _ops().linear_gelu(x, weight, bias)


def linear_dropout_add(x: torch.Tensor, weight: torch.Tensor, bias, residual: torch.Tensor,
                       p: float = 0.1, training: bool = True, seed: int | None = None,
                       stream: int | None = None, generator: str = "philox4x32") -> torch.Tensor:
    """``residual + dropout(linear(x))`` as one node (a transformer block's
    output projection before its LayerNorm).

    ``torch.ops.memsave.linear_dropout_add`` (``LinearDropoutAddFn``) applies
    the dropout and the residual add in the GEMM epilogue; every intermediate is
    rounded as the separate launches round it and the mask is the one
    :func:`dropout` draws for the same (seed, stream), so values equal the
    three ops.  Saved set: the Linear's rule (rules.py:133-141) and the
    dropout's RNG key (rules.py:103-106); the add keeps nothing.  ``stream``
    defaults to DROPOUT_STREAM_BASE like :func:`dropout`."""
    if not 0.0 <= p < 1.0:
        raise ValueError(f"dropout probability has to be in [0, 1), got {p}")
    if generator not in _RNG:
        raise ValueError(f"dropout generator must be one of {sorted(_RNG)}, got {generator!r}")
    pe = float(p) if training else 0.0
    sd = (draw_seed() if seed is None else int(seed)) if pe > 0.0 else 0
    return _ops().linear_dropout_add(x, weight, bias, residual, pe, sd,
                                     DROPOUT_STREAM_BASE if stream is None else int(stream),
                                     _RNG[generator])


# =============================================================== conv2d
def _pair(v):
    if isinstance(v, (tuple, list)):
        return int(v[0]), int(v[1])
    return int(v), int(v)


def _conv_layouts(x: torch.Tensor, weight: torch.Tensor):
    """Pick activation / weight layouts.  16-bit activations always run NHWC
    (the tcgen05 implicit-GEMM path); float32 keeps the caller's layout."""
    if x.dtype in (torch.bfloat16, torch.float16):
        layout = _lib.MS_NHWC
    else:
        layout = _lib.MS_NHWC if (_is_channels_last(x) and not x.is_contiguous()) else _lib.MS_NCHW
    if weight.is_contiguous(memory_format=torch.channels_last):
        wlayout = _lib.MS_NHWC
    else:
        wlayout = _lib.MS_NCHW
    return layout, wlayout


def _as_layout(t: torch.Tensor, layout: int) -> torch.Tensor:
    if layout == _lib.MS_NHWC:
        return t.contiguous(memory_format=torch.channels_last)
    return t.contiguous()


def _check_conv_channels(x_shape, w_shape) -> None:
    if w_shape[1] != x_shape[1]:
        raise RuntimeError(f"conv2d: input channels {x_shape[1]} != weight channels {w_shape[1]} "
                           f"(groups unsupported)")


def _conv_out_hw(x_shape, w_shape, stride, padding):
    oh = (x_shape[2] + 2 * padding[0] - w_shape[2]) // stride[0] + 1
    ow = (x_shape[3] + 2 * padding[1] - w_shape[3]) // stride[1] + 1
    if oh <= 0 or ow <= 0:
        raise RuntimeError(f"conv2d: empty output for input {tuple(x_shape)} / kernel "
                           f"{tuple(w_shape)}")
    return oh, ow


class _Conv2dFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, stride, padding):
        x_rg, w_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        roles = saved_roles(x_rg, w_rg)
        stride, padding = _pair(stride), _pair(padding)
        if x.dim() != 4 or weight.dim() != 4:
            raise RuntimeError("conv2d: expected 4-d input (N, C, H, W) and weight (K, C, R, S)")
        oh, ow = _conv_out_hw(x.shape, weight.shape, stride, padding)
        ctx.geom = (tuple(x.shape), tuple(weight.shape), stride, padding)
        ctx.w_meta = (weight.dtype, weight.is_contiguous(memory_format=torch.channels_last)
                      and not weight.is_contiguous())
        out_shape = (x.shape[0], weight.shape[0], oh, ow)
        if _is_meta(x, weight):
            ctx.save_for_backward(x if "x" in roles else None, weight if "w" in roles else None)
            ctx.layouts = (_lib.MS_NCHW, _lib.MS_NCHW)
            return x.new_empty(out_shape)
        _require_cuda("conv2d", x, weight, bias)
        if weight.dtype != x.dtype:
            raise TypeError(f"conv2d: input dtype {x.dtype} != weight dtype {weight.dtype}")
        layout, wlayout = _conv_layouts(x, weight)
        xl = _as_layout(x, layout)
        wl = _as_layout(weight, wlayout)
        ctx.layouts = (layout, wlayout)
        ctx.save_for_backward(xl if "x" in roles else None, wl if "w" in roles else None)
        _dtype_code(x)
        _check_conv_channels(x.shape, weight.shape)
        return _ops().conv2d_fwd(xl, wl, bias, list(stride), list(padding), layout, wlayout)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        need_x, need_w, need_b = ctx.needs_input_grad[:3]
        x_shape, w_shape, stride, padding = ctx.geom
        w_dtype, w_cl = ctx.w_meta
        dx = dw = db = None
        if _is_meta(gy):
            # mirror the CUDA path's allocations (the planner's ledger sees them):
            # an expanded upstream gradient is materialised in the kernel layout
            gy = _as_layout(gy, ctx.layouts[0])
            if need_x:
                _need(w, "w", "conv2d dX")
                dx = gy.new_empty(x_shape)
            if need_w:
                _need(x, "x", "conv2d dW")
                dw = gy.new_empty(w_shape)
            if need_b:
                db = gy.new_empty((w_shape[0],))
            return dx, dw, db, None, None
        layout, wlayout = ctx.layouts
        g = _as_layout(gy, layout)
        O = _ops()
        geo = (list(stride), list(padding), layout, wlayout)
        if need_x:
            w = _need(w, "w", "conv2d dX")
            dx = O.conv2d_dx(g, w, list(x_shape), *geo)
        if need_w:
            x = _need(x, "x", "conv2d dW")
            dw = O.conv2d_dw(x, g, list(w_shape), *geo)
        if need_b:
            db = O.conv2d_db(g, list(x_shape), list(w_shape), *geo)
        return dx, dw, db, None, None


def conv2d(x, weight, bias=None, stride=1, padding=0):
    """Differentiability-agnostic 2-d cross-correlation."""
    return _Conv2dFn.apply(x, weight, bias, stride, padding)


# =============================================================== batchnorm2d (eval)
class _BatchNorm2dEvalFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, running_mean, running_var, eps):
        x_rg, w_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        roles = saved_roles(x_rg, w_rg)
        # Running statistics are module state, not tape state:
        # they are referenced from ctx, never passed to save_for_backward.
        ctx.stats = (running_mean, running_var)
        ctx.eps = float(eps)
        ctx.x_shape = tuple(x.shape)
        ctx.p_dtypes = (None if weight is None else weight.dtype,
                        None if bias is None else bias.dtype)
        if x.dim() != 4:
            raise RuntimeError("batchnorm2d: expected a 4-d input")
        if _is_meta(x):
            ctx.layout = _lib.MS_NCHW
            ctx.save_for_backward(x if "x" in roles else None, weight if "w" in roles else None)
            return x.new_empty(x.shape)
        _require_cuda("batch_norm", x, weight, bias, running_mean, running_var)
        layout = _lib.MS_NHWC if (_is_channels_last(x) and not x.is_contiguous()) else _lib.MS_NCHW
        xl = _as_layout(x, layout)
        ctx.layout = layout
        ctx.save_for_backward(xl if "x" in roles else None, weight if "w" in roles else None)
        _dtype_code(x)
        return _ops().bn_eval_fwd(xl, running_mean, running_var, weight, bias, ctx.eps, layout)

    @staticmethod
    def backward(ctx, gy):
        x, weight = ctx.saved_tensors
        need_x, need_w, need_b = ctx.needs_input_grad[:3]
        running_mean, running_var = ctx.stats
        c = ctx.x_shape[1]
        dx = dw = db = None
        if _is_meta(gy):
            if need_x:
                dx = gy.new_empty(ctx.x_shape)
            if need_w:
                _need(x, "x", "batchnorm2d dW")
                dw = gy.new_empty((c,))
            if need_b:
                db = gy.new_empty((c,))
            return dx, dw, db, None, None, None
        if need_x and ctx.p_dtypes[0] is not None:
            weight = _need(weight, "w", "batchnorm2d dX")
        if need_w:
            x = _need(x, "x", "batchnorm2d dW")
        layout = ctx.layout
        g = _as_layout(gy, layout)
        # dW and db come back as the two rows of one [2, C] statistics-dtype buffer
        dx_t, dwdb = _ops().bn_eval_bwd(g, x if need_w else None, running_mean, running_var,
                                        weight, ctx.eps, layout, bool(need_x), bool(need_w),
                                        bool(need_b))
        dx = _opt(dx_t, need_x)
        if need_w:
            dw = dwdb[0].to(ctx.p_dtypes[0])
        if need_b:
            db = dwdb[1].to(ctx.p_dtypes[1])
        return dx, dw, db, None, None, None


class _BatchNorm2dEvalReLUFn(torch.autograd.Function):
    """BatchNorm2d(eval) -> ReLU in one pass (ms_bn_eval_relu_fwd), for BN layers
    with a trainable affine (which the conv epilogue cannot absorb).  Saved set
    = the union of the two rows: x iff the BN weight needs a grad, the weight
    iff x does (rules.py:84-87 linear family), the ReLU bit mask iff the output
    needs a grad (rules.py:98-101).  Backward: one pass for keep * (BN VJP).

    ``residual`` (optional): relu(bn(x) + residual), a bottleneck block's tail
    (the add saves nothing, rules.py:116-117); its gradient g * keep is written
    by the same backward pass (ms_bn_eval_add_relu_{fwd,bwd})."""

    @staticmethod
    def forward(ctx, x, weight, bias, running_mean, running_var, eps, residual=None):
        x_rg, w_rg, b_rg = ctx.needs_input_grad[:3]
        roles = saved_roles(x_rg, w_rg)
        out_rg = x_rg or w_rg or b_rg or ctx.needs_input_grad[6]
        ctx.stats = (running_mean, running_var)
        ctx.eps = float(eps)
        ctx.x_shape = tuple(x.shape)
        ctx.p_dtypes = (None if weight is None else weight.dtype,
                        None if bias is None else bias.dtype)
        n_el = x.numel()
        if _is_meta(x):
            mask = torch.empty((n_el + 7) // 8, dtype=torch.uint8, device="meta") if out_rg \
                else None
            ctx.save_for_backward(x if "x" in roles else None, weight if "w" in roles else None,
                                  mask)
            return x.new_empty(x.shape)
        _require_cuda("batch_norm_relu", x, weight, bias, running_mean, running_var)
        xl = _as_layout(x, _lib.MS_NHWC)
        rl = None
        if residual is not None:
            _require_cuda("batch_norm_add_relu", residual)
            if residual.shape != x.shape or residual.dtype != x.dtype:
                raise RuntimeError("bn+add+relu: residual must match the BN input's shape "
                                   "and dtype")
            rl = _as_layout(residual, _lib.MS_NHWC)
        y, mask = _ops().bn_relu_fwd(xl, rl, running_mean, running_var, weight, bias, ctx.eps,
                                     bool(out_rg))
        mask = _opt(mask, out_rg)
        ctx.save_for_backward(xl if "x" in roles else None, weight if "w" in roles else None,
                              mask)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, weight, mask = ctx.saved_tensors
        need_x, need_w, need_b = ctx.needs_input_grad[:3]
        need_r = ctx.needs_input_grad[6]
        running_mean, running_var = ctx.stats
        c = ctx.x_shape[1]
        mask = _need(mask, "mask", "batchnorm2d+relu backward")
        dx = dw = db = dr = None
        if _is_meta(gy):
            if need_x:
                dx = gy.new_empty(ctx.x_shape)
            if need_w:
                _need(x, "x", "batchnorm2d dW")
                dw = gy.new_empty((c,))
            if need_b:
                db = gy.new_empty((c,))
            if need_r:
                dr = gy.new_empty(ctx.x_shape)
            return dx, dw, db, None, None, None, dr
        if need_x and ctx.p_dtypes[0] is not None:
            weight = _need(weight, "w", "batchnorm2d dX")
        if need_w:
            x = _need(x, "x", "batchnorm2d dW")
        g = _as_layout(gy, _lib.MS_NHWC)
        dx_t, dr_t, dwdb = _ops().bn_add_relu_bwd(g, mask, x if need_w else None, running_mean,
                                                  running_var, weight, ctx.eps, bool(need_x),
                                                  bool(need_r), bool(need_w), bool(need_b))
        dx, dr = _opt(dx_t, need_x), _opt(dr_t, need_r)
        if need_w:
            dw = dwdb[0].to(ctx.p_dtypes[0])
        if need_b:
            db = dwdb[1].to(ctx.p_dtypes[1])
        return dx, dw, db, None, None, None, dr


def bn_relu_fusable(x: torch.Tensor, bn) -> bool:
    """The one-pass BN-eval -> ReLU kernel applies (any requires_grad of the affine)."""
    if bn is None or bn.training or not bn.track_running_stats or bn.running_var is None:
        return False
    if x.dim() != 4 or x.shape[1] % 8 or x.shape[1] > 2048:
        return False
    if x.device.type == "meta":
        return x.dtype in (torch.bfloat16, torch.float16)
    return x.device.type == "cuda" and x.dtype in (torch.bfloat16, torch.float16) \
        and _is_channels_last(x)


def batch_norm_relu_eval(x, bn, residual=None):
    """relu(bn(x) [+ residual]) for an eval-mode BatchNorm2d module in one pass."""
    return _BatchNorm2dEvalReLUFn.apply(x, bn.weight, bn.bias, bn.running_mean, bn.running_var,
                                        bn.eps, residual)


def batch_norm_eval(x, running_mean, running_var, weight=None, bias=None, eps=1e-5):
    """Differentiability-agnostic eval-mode batch norm."""
    return _BatchNorm2dEvalFn.apply(x, weight, bias, running_mean, running_var, eps)


# =============================================================== relu (bit mask)
def _dense_format(t: torch.Tensor):
    """Memory format in which ``t`` is dense (the mask follows storage order)."""
    if t.is_contiguous():
        return torch.contiguous_format
    if _is_channels_last(t):
        return torch.channels_last
    return None


class _ReLUFn(torch.autograd.Function):
    """MemSave ReLU (rules.py:98-101, MEMSAVE row): keeps a bit-packed mask of
    x > 0 (saved.py:53-71, ceil(numel/8) bytes) instead of the output tensor."""

    @staticmethod
    def forward(ctx, x, inplace: bool):
        x_rg = ctx.needs_input_grad[0]
        if _is_meta(x):
            ctx.save_for_backward(torch.empty((x.numel() + 7) // 8, dtype=torch.uint8,
                                              device="meta") if x_rg else None)
            ctx.fmt = torch.contiguous_format
            return x.new_empty(x.shape)
        _require_cuda("relu", x)
        fmt = _dense_format(x)
        if fmt is None:
            x = x.contiguous()
            fmt = torch.contiguous_format
            inplace = False
        ctx.fmt = fmt
        _dtype_code(x)
        if inplace:
            mask = _ops().relu_fwd_(x, bool(x_rg))
            y = x
            ctx.mark_dirty(x)
        else:
            y, mask = _ops().relu_fwd(x, bool(x_rg))
        ctx.save_for_backward(_opt(mask, x_rg))
        return y

    @staticmethod
    def backward(ctx, gy):
        (mask,) = ctx.saved_tensors
        if not ctx.needs_input_grad[0]:
            return None, None
        mask = _need(mask, "mask", "relu dX")
        if _is_meta(gy):
            gy = gy.contiguous(memory_format=ctx.fmt)  # mirrors the CUDA path's allocation
            return gy.new_empty(gy.shape), None
        g = gy.contiguous(memory_format=ctx.fmt)
        return _ops().relu_bwd(g, mask), None


def relu(x: torch.Tensor, inplace: bool = False) -> torch.Tensor:
    """ReLU whose backward reads a 1-bit mask (SPEC.md forward_relu, Masked)."""
    return _ReLUFn.apply(x, inplace)


# =============================================================== maxpool2d (index map)
class _MaxPool2dFn(torch.autograd.Function):
    """MemSave MaxPool2d: keeps a 1-byte window-local argmax per output element
    (rules.py:108-109; the reference's IndexMap, saved.py:111-125, is 4 bytes)."""

    @staticmethod
    def forward(ctx, x, kernel_size, stride, padding, in_mask=None, in_bn=None):
        # in_mask / in_bn: x came out of a fused ReLU [after eval-BN]; its backward
        # (keep [* s]) is applied in this backward's store (ms_maxpool2d_relu_bwd)
        if in_mask is None:
            in_bn = None
        ctx.in_bn = None if in_bn is None else (in_bn.running_mean, in_bn.running_var,
                                                in_bn.weight, float(in_bn.eps))
        kh, kw = _pair(kernel_size)
        sh, sw = _pair(stride)
        ph, pw = _pair(padding)
        x_rg = ctx.needs_input_grad[0]
        if x.dim() != 4:
            raise RuntimeError("max_pool2d: expected a 4-d input")
        n, c, h, w = x.shape
        oh = (h + 2 * ph - kh) // sh + 1
        ow = (w + 2 * pw - kw) // sw + 1
        ctx.geom = (tuple(x.shape), kh, kw, sh, sw, ph, pw)
        keep = in_mask if x_rg else None
        if _is_meta(x):
            ctx.layout = _lib.MS_NCHW
            ctx.save_for_backward(torch.empty((n, c, oh, ow), dtype=torch.uint8, device="meta")
                                  if x_rg else None, keep)
            return x.new_empty((n, c, oh, ow))
        _require_cuda("max_pool2d", x)
        layout = _lib.MS_NHWC if (_is_channels_last(x) and not x.is_contiguous()) else _lib.MS_NCHW
        xl = _as_layout(x, layout)
        ctx.layout = layout
        _dtype_code(x)
        y, idx = _ops().maxpool2d_fwd(xl, [kh, kw], [sh, sw], [ph, pw], layout, bool(x_rg))
        ctx.save_for_backward(_opt(idx, x_rg), keep)
        return y

    @staticmethod
    def backward(ctx, gy):
        idx, keep = ctx.saved_tensors
        nones = (None,) * 5
        if not ctx.needs_input_grad[0]:
            return (None,) + nones
        idx = _need(idx, "idx", "max_pool2d dX")
        x_shape, kh, kw, sh, sw, ph, pw = ctx.geom
        if _is_meta(gy):
            return (gy.new_empty(x_shape),) + nones
        layout = ctx.layout
        g = _as_layout(gy, layout)
        geo = (list(x_shape), [kh, kw], [sh, sw], [ph, pw], layout)
        if keep is not None:
            # the producer ReLU [+ eval-BN]'s backward applied at the pool's store
            ib = ctx.in_bn or (None, None, None, 0.0)
            return (_ops().maxpool2d_relu_bwd(g, idx, keep, ib[0], ib[1], ib[2], ib[3], *geo),) \
                + nones
        return (_ops().maxpool2d_bwd(g, idx, *geo),) + nones


def max_pool2d(x, kernel_size, stride=None, padding=0, in_mask=None, in_bn=None):
    """Max pooling whose backward reads a 1-byte argmax map (SPEC.md forward_maxpool2d).
    ``in_mask`` / ``in_bn``: x is the raw output of a fused conv -> [BN ->] ReLU
    (fused_conv(raw=True)); the ReLU [+ BN scale] backward then runs in this
    backward's store."""
    return _MaxPool2dFn.apply(x, kernel_size, kernel_size if stride is None else stride, padding,
                              in_mask, in_bn)


# =============================================================== dropout (RNG replay)
DROPOUT_STREAM_BASE = 1_000_000  # leantape.core.Rng.DROPOUT_STREAM_BASE (core.py:108)
# mask generators (include/memsave_b200.h ms_rng): "philox4x32" (default, Random123
# Philox4x32-10) or "reference" (leantape.core.Rng's Philox4x64-10, bit-identical
# to the reference's masks)
_RNG = {"philox4x32": _lib.MS_RNG_PHILOX4X32, "reference": _lib.MS_RNG_PHILOX4X64_REF}


class _DropoutFn(torch.autograd.Function):
    """MemSave Dropout (rules.py:103-106, MEMSAVE row): keeps only the 16-byte
    RNG key (seed, stream) (saved.py:91-108, RngSeed) and regenerates the keep
    mask in backward from the counter-based generator ``gen`` (with
    "reference", Rng(seed, stream).uniform() >= p of core.py:100-124)."""

    @staticmethod
    def forward(ctx, x, p: float, seed: int, stream: int, inplace: bool, gen: int):
        out_rg = ctx.needs_input_grad[0]
        ctx.key = (int(seed), int(stream), float(p), int(gen))
        key = torch.tensor([int(seed), int(stream)], dtype=torch.int64) if out_rg else None
        if _is_meta(x):
            ctx.save_for_backward(key)
            return x.new_empty(x.shape)
        _require_cuda("dropout", x)
        fmt = _dense_format(x)
        if fmt is None:
            x = x.contiguous()
            fmt = torch.contiguous_format
            inplace = False
        ctx.fmt = fmt
        _dtype_code(x)
        if inplace:
            _ops().dropout_fwd_(x, p, seed, stream, gen)
            y = x
            ctx.mark_dirty(x)
        else:
            y = _ops().dropout_fwd(x, p, seed, stream, gen)
        ctx.save_for_backward(key)
        return y

    @staticmethod
    def backward(ctx, gy):
        (key,) = ctx.saved_tensors
        if not ctx.needs_input_grad[0]:
            return None, None, None, None, None, None
        _need(key, "seed", "dropout dX")
        seed, stream, p, gen = ctx.key
        if _is_meta(gy):
            gy = gy.contiguous()  # mirrors the CUDA path's allocation
            return gy.new_empty(gy.shape), None, None, None, None, None
        g = gy.contiguous(memory_format=ctx.fmt)
        return _ops().dropout_bwd(g, p, seed, stream, gen), None, None, None, None, None


def draw_seed() -> int:
    """A fresh 62-bit dropout seed from torch's default CPU generator (so
    ``torch.manual_seed`` makes runs reproducible)."""
    return int(torch.randint(0, 2 ** 62, (1,)).item())


def dropout(x: torch.Tensor, p: float = 0.5, training: bool = True, inplace: bool = False,
            seed: int | None = None, stream: int = DROPOUT_STREAM_BASE,
            generator: str = "philox4x32") -> torch.Tensor:
    """Dropout whose backward replays the mask from its RNG key (SPEC.md
    forward_dropout, RngReplay variant).  ``generator="reference"`` draws the
    reference's own masks (leantape.core.Rng); seeds must be < 2^63."""
    if not 0.0 <= p < 1.0:
        raise ValueError(f"dropout probability has to be in [0, 1), got {p}")
    if generator not in _RNG:
        raise ValueError(f"dropout generator must be one of {sorted(_RNG)}, got {generator!r}")
    if not training or p == 0.0:
        return x
    return _DropoutFn.apply(x, float(p), draw_seed() if seed is None else int(seed), int(stream),
                            inplace, _RNG[generator])


# =============================================================== layernorm
class _LayerNormFn(torch.autograd.Function):
    """LayerNorm over the trailing ``normalized_shape`` dims (rules.py:89-96,
    identical under both policies): keeps x and the per-row (mean, rstd) iff x
    or w needs a gradient, and w iff x does; db reads nothing."""

    @staticmethod
    def forward(ctx, x, normalized_shape, weight, bias, eps):
        x_rg, w_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[2]
        nshape = tuple(int(s) for s in normalized_shape)
        if tuple(x.shape[x.dim() - len(nshape):]) != nshape:
            raise RuntimeError(f"layer_norm: input {tuple(x.shape)} does not end with {nshape}")
        dim = 1
        for s in nshape:
            dim *= s
        rows = x.numel() // dim if dim else 0
        ctx.dims = (rows, dim, tuple(x.shape))
        ctx.nshape = nshape
        ctx.p_dtypes = (None if weight is None else weight.dtype,
                        None if bias is None else bias.dtype)
        keep_x = x_rg or w_rg
        if _is_meta(x):
            mean = torch.empty(rows, dtype=torch.float32, device="meta") if keep_x else None
            rstd = torch.empty(rows, dtype=torch.float32, device="meta") if keep_x else None
            ctx.save_for_backward(x if keep_x else None, mean, rstd, weight if x_rg else None)
            return x.new_empty(x.shape)
        _require_cuda("layer_norm", x, weight, bias)
        _dtype_code(x)
        xc = x.contiguous()
        w = None if weight is None else weight.to(x.dtype).contiguous()
        y, mean, rstd = _ops().layernorm_fwd(xc, w, bias, float(eps), dim, bool(keep_x))
        ctx.save_for_backward(xc if keep_x else None, _opt(mean, keep_x), _opt(rstd, keep_x),
                              w if x_rg else None)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, mean, rstd, w = ctx.saved_tensors
        need_x, need_w, need_b = (ctx.needs_input_grad[0], ctx.needs_input_grad[2],
                                  ctx.needs_input_grad[3])
        rows, dim, shape = ctx.dims
        w_dt, b_dt = ctx.p_dtypes
        dx = dw = db = None
        if _is_meta(gy):
            if need_x:
                _need(x, "x", "layer_norm dX")
                dx = gy.new_empty(shape)
            if need_w:
                _need(x, "x", "layer_norm dW")
                dw = torch.empty(ctx.nshape, dtype=w_dt, device="meta")
            if need_b:
                db = torch.empty(ctx.nshape, dtype=b_dt, device="meta")
            return dx, None, dw, db, None
        g = gy.contiguous()
        if need_x or need_w:
            x = _need(x, "x", "layer_norm dX/dW")
            _need(mean, "stats", "layer_norm dX/dW")
            if need_x and ctx.p_dtypes[0] is not None:
                _need(w, "w", "layer_norm dX")
            dxt, dwt, dbt = _ops().layernorm_bwd(g, x, mean, rstd, w, dim, bool(need_x),
                                                 bool(need_w), bool(need_b))
            dx, dw, db = _opt(dxt, need_x), _opt(dwt, need_w), _opt(dbt, need_b)
        elif need_b:  # db = sum_rows g: nothing saved is read
            db = _ops().bias_grad(g, dim)
        if dw is not None:
            dw = dw.view(ctx.nshape).to(w_dt)
        if db is not None:
            db = db.view(ctx.nshape).to(b_dt)
        if dx is not None:
            dx = dx.view(shape)
        return dx, None, dw, db, None


def layer_norm(x, normalized_shape, weight=None, bias=None, eps: float = 1e-5):
    """``F.layer_norm`` on the sm_100a kernels (SPEC.md forward_layernorm)."""
    if isinstance(normalized_shape, int):
        normalized_shape = (normalized_shape,)
    return _LayerNormFn.apply(x, tuple(normalized_shape), weight, bias, eps)


# =============================================================== conv_transpose2d
class _ConvTranspose2dFn(torch.autograd.Function):
    """ConvTranspose2d (rules.py:68-71, MEMSAVE row = linear family; SPEC.md
    forward_conv_transpose2d).  Its forward is the input-VJP of the conv2d
    whose weight it shares ([C_in][C_out][kh][kw] = conv [K][C][R][S]), its dX
    is that conv's forward and its dW the conv's weight-VJP with the operand
    roles swapped, so it runs on the same kernels (ms_conv2d_dx / _fwd / _dw)."""

    @staticmethod
    def forward(ctx, x, weight, bias, stride, padding, output_padding):
        x_rg, w_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        roles = saved_roles(x_rg, w_rg)
        stride, padding, opad = _pair(stride), _pair(padding), _pair(output_padding)
        if x.dim() != 4 or weight.dim() != 4:
            raise RuntimeError("conv_transpose2d: expected 4-d input and weight")
        n, cin, h, w_ = x.shape
        if weight.shape[0] != cin:
            raise RuntimeError(f"conv_transpose2d: input channels {cin} != weight.shape[0] "
                               f"{weight.shape[0]} (groups unsupported)")
        cout, kh, kw = weight.shape[1], weight.shape[2], weight.shape[3]
        ho = (h - 1) * stride[0] - 2 * padding[0] + kh + opad[0]
        wo = (w_ - 1) * stride[1] - 2 * padding[1] + kw + opad[1]
        if ho <= 0 or wo <= 0 or opad[0] >= max(stride[0], 1) or opad[1] >= max(stride[1], 1):
            raise RuntimeError("conv_transpose2d: invalid output size / output_padding")
        # the equivalent conv2d: input (n, cout, ho, wo) -> output (n, cin, h, w)
        conv_x = (n, cout, ho, wo)
        ctx.geom = (conv_x, tuple(weight.shape), stride, padding, tuple(x.shape))
        ctx.w_meta = weight.dtype
        if _is_meta(x, weight):
            ctx.save_for_backward(x if "x" in roles else None, weight if "w" in roles else None)
            ctx.layouts = (_lib.MS_NCHW, _lib.MS_NCHW)
            return x.new_empty(conv_x)
        _require_cuda("conv_transpose2d", x, weight, bias)
        if weight.dtype != x.dtype:
            raise TypeError(f"conv_transpose2d: input dtype {x.dtype} != weight dtype "
                            f"{weight.dtype}")
        layout, wlayout = _conv_layouts(x, weight)
        xl = _as_layout(x, layout)
        wl = _as_layout(weight, wlayout)
        ctx.layouts = (layout, wlayout)
        ctx.save_for_backward(xl if "x" in roles else None, wl if "w" in roles else None)
        _dtype_code(x)
        return _ops().conv_transpose2d_fwd(xl, wl, bias, list(conv_x), list(stride),
                                           list(padding), layout, wlayout)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        need_x, need_w, need_b = ctx.needs_input_grad[:3]
        conv_x, w_shape, stride, padding, x_shape = ctx.geom
        dx = dw = db = None
        if _is_meta(gy):
            if need_x:
                _need(w, "w", "conv_transpose2d dX")
                dx = gy.new_empty(x_shape)
            if need_w:
                _need(x, "x", "conv_transpose2d dW")
                dw = gy.new_empty(w_shape)
            if need_b:
                db = gy.new_empty((w_shape[1],))
            return dx, dw, db, None, None, None
        layout, wlayout = ctx.layouts
        g = _as_layout(gy, layout)
        O = _ops()
        geo = (list(stride), list(padding), layout, wlayout)
        if need_x:  # dX = conv2d(g, W)
            w = _need(w, "w", "conv_transpose2d dX")
            dx = O.conv2d_fwd(g, w, None, *geo)
        if need_w:  # dW = conv2d weight-VJP with the conv input g and conv output-grad x
            x = _need(x, "x", "conv_transpose2d dW")
            dw = O.conv2d_dw(g, x, list(w_shape), *geo)
        if need_b:  # sum of g over (n, h, w) per output channel
            c = conv_x[1]
            db = O.conv2d_db(g, list(conv_x), [c, c, 1, 1], [1, 1], [0, 0], layout, wlayout)
        return dx, dw, db, None, None, None


def conv_transpose2d(x, weight, bias=None, stride=1, padding=0, output_padding=0):
    """Differentiability-agnostic ``F.conv_transpose2d`` (groups = dilation = 1)."""
    return _ConvTranspose2dFn.apply(x, weight, bias, stride, padding, output_padding)


# =============================================================== fused conv -> BN-eval (-> ReLU)
def _bn_frozen_eval(bn) -> bool:
    return (not bn.training and bn.running_mean is not None and bn.running_var is not None
            and not any(p.requires_grad for p in bn.parameters()))


class _ConvBNFn(torch.autograd.Function):
    """conv2d -> BatchNorm2d(eval, frozen) [-> ReLU] in one tcgen05 launch (BN affine
    and ReLU in the conv epilogue).  Saved set = the union of the three layers'
    rows: W iff x needs a grad and x iff W needs one (rules.py:68-71, MEMSAVE),
    nothing for the frozen eval-BN (rules.py:84-87), the ReLU bit mask iff the
    output needs a grad (rules.py:98-101; kept by _MaskScaleFn, which also
    applies it).  Returns (y, mask).  Backward gets dL/d(conv * s): with a ReLU
    that is the masked, scaled gradient from _MaskScaleFn; without one the BN
    scale is folded into the dgrad weight (dX = dgrad(g, W * s)) so the large
    gradient is never rescaled."""

    @staticmethod
    def forward(ctx, x, weight, bias, residual, stride, padding, bn, relu: bool, tee=False,
                in_mask=None, in_bn=None):
        # tee: also return x itself, for x's other consumer; backward then adds that
        # consumer's gradient in the dgrad epilogue instead of the engine summing it.
        # in_mask / in_bn: x came out of a fused ReLU [after eval-BN in_bn] whose
        # backward (keep mask [and BN scale]) runs in this node's dgrad epilogue.
        x_rg, w_rg, b_rg = ctx.needs_input_grad[0], ctx.needs_input_grad[1], ctx.needs_input_grad[2]
        ctx.tee = bool(tee)
        if in_mask is None:
            in_bn = None
        ctx.in_bn = None if in_bn is None else (in_bn.running_mean, in_bn.running_var,
                                                in_bn.weight, float(in_bn.eps))
        keep = in_mask if x_rg else None  # the ReLU mask rule (rules.py:98-101), kept here
        out_rg = x_rg or w_rg or b_rg or ctx.needs_input_grad[3]
        ctx.set_materialize_grads(False)  # the mask output never gets a gradient: no zero fill
        # the incoming gradient is already masked and scaled (_MaskScaleFn) only for
        # conv -> BN -> ReLU without a residual; otherwise the BN scale is folded here
        ctx.prescaled = bool(relu) and residual is None and bn is not None
        roles = saved_roles(x_rg, w_rg)
        stride, padding = _pair(stride), _pair(padding)
        oh, ow = _conv_out_hw(x.shape, weight.shape, stride, padding)
        ctx.geom = (tuple(x.shape), tuple(weight.shape), stride, padding)
        ctx.w_meta = (weight.dtype, False)
        ctx.bn = None if bn is None else (bn.running_mean, bn.running_var, bn.weight,
                                          float(bn.eps))
        ctx.relu = bool(relu)
        out_shape = (x.shape[0], weight.shape[0], oh, ow)
        n_el = x.shape[0] * weight.shape[0] * oh * ow
        if _is_meta(x, weight):
            mask = (torch.empty((n_el + 7) // 8, dtype=torch.uint8, device="meta")
                    if relu and out_rg else None)
            ctx.save_for_backward(x if "x" in roles else None, weight if "w" in roles else None,
                                  keep)
            ctx.layouts = (_lib.MS_NCHW, _lib.MS_NCHW)
            if mask is not None:
                ctx.mark_non_differentiable(mask)
            return (x.new_empty(out_shape), mask, x) if tee else (x.new_empty(out_shape), mask)
        _require_cuda("conv_bn", x, weight, bias)
        layout, wlayout = _conv_layouts(x, weight)
        xl = _as_layout(x, layout)
        wl = _as_layout(weight, wlayout)
        ctx.layouts = (layout, wlayout)
        _dtype_code(x)
        _check_conv_channels(x.shape, weight.shape)
        res = None if residual is None else _as_layout(residual, layout)
        mean, var, bw, eps = ctx.bn if bn is not None else (None, None, None, 0.0)
        bb = None if bn is None else bn.bias
        y, mask = _ops().conv2d_bn_fwd(xl, wl, bias, mean, var, bw, bb, eps, res, bool(relu),
                                       bool(out_rg), list(stride), list(padding), layout, wlayout)
        mask = _opt(mask, relu and out_rg)
        ctx.save_for_backward(xl if "x" in roles else None, wl if "w" in roles else None, keep)
        if mask is not None:
            ctx.mark_non_differentiable(mask)
        return (y, mask, x) if tee else (y, mask)

    @staticmethod
    def backward(ctx, gy, _gmask=None, g_tee=None):
        x, w, keep = ctx.saved_tensors
        nones = (None,) * 10
        if gy is None:  # grads are not materialised (set_materialize_grads(False))
            if g_tee is None or not ctx.needs_input_grad[0]:
                return (None,) + nones
            if keep is None:
                return (g_tee,) + nones
            # the keep mask follows the kernel layout's element order (channel = idx % C)
            return (_mask_scale(_as_layout(g_tee, ctx.layouts[0]), keep, ctx.in_bn),) + nones
        need_x, need_w, need_b = ctx.needs_input_grad[:3]
        x_shape, w_shape, stride, padding = ctx.geom
        dx = dw = db = None
        layout, wlayout = ctx.layouts
        mean, var, bw, eps = ctx.bn if ctx.bn is not None else (None, None, None, 0.0)
        g = _as_layout(gy, layout)
        del gy
        addend = _as_layout(g_tee, layout) if (need_x and g_tee is not None) else None
        del g_tee
        need_r = ctx.needs_input_grad[3]
        d_res = g if need_r else None  # the residual's gradient is the (masked) gradient
        if ctx.bn is None:  # conv [-> relu]: g (masked by _MaskScaleFn) is dL/dconv
            sc_w = False
            need_scaled_g = False
        elif not ctx.prescaled:
            # dL/dconv = g * s: fold s into W for dX; scale g only for dW / db
            sc_w = need_x
            need_scaled_g = need_w or need_b
        else:
            sc_w = False  # g arrives already masked and scaled (_MaskScaleFn)
            need_scaled_g = False
        if _is_meta(g):  # mirror the CUDA path's allocations for the planner
            gc = torch.empty_like(g) if need_scaled_g else g
            if need_x:
                _need(w, "w", "conv_bn dX")
                dx = gc.new_empty(x_shape)
            if need_w:
                _need(x, "x", "conv_bn dW")
                dw = gc.new_empty(w_shape)
            if need_b:
                db = gc.new_empty((w_shape[0],))
            return (dx, dw, db, d_res) + (None,) * 7
        O = _ops()
        geo = (list(stride), list(padding), layout, wlayout)
        if need_x:
            w = _need(w, "w", "conv_bn dX")
            ib = ctx.in_bn or (None, None, None, 0.0)
            if sc_w or addend is not None or keep is not None:
                # BN scale folded into the repacked dgrad weight (no pass over g), the
                # tee'd consumer's gradient and the producer ReLU [+BN]'s backward in
                # the epilogue (the op runs the separate passes where it cannot)
                dx = O.conv2d_bn_dx(g, w, var if sc_w else None, bw if sc_w else None, eps,
                                    addend, keep, ib[0], ib[1], ib[2], ib[3], list(x_shape), *geo)
            else:
                dx = O.conv2d_dx(g, w, list(x_shape), *geo)
            del addend
        if need_w or need_b:
            gc = O.bn_relu_bwd(g, None, mean, var, bw, eps) if need_scaled_g else g
            if need_w:
                x = _need(x, "x", "conv_bn dW")
                dw = O.conv2d_dw(x, gc, list(w_shape), *geo)
            if need_b:
                db = O.conv2d_db(gc, list(x_shape), list(w_shape), *geo)
        return (dx, dw, db, d_res) + (None,) * 7


def _mask_scale(g: torch.Tensor, keep: torch.Tensor, bnp) -> torch.Tensor:
    """g * keep [* s] as its own pass (ms_relu_bwd / ms_bn_relu_bwd): the fallback
    of the ReLU [+ eval-BN] backward that a fused dgrad epilogue normally applies."""
    keep = _need(keep, "mask", "ReLU backward")
    fmt = torch.channels_last if _is_channels_last(g) and not g.is_contiguous() \
        else torch.contiguous_format
    g = g.contiguous(memory_format=fmt)
    if _is_meta(g):
        return torch.empty_like(g, memory_format=fmt)
    if bnp is None:
        return _ops().relu_bwd(g, keep)
    mean, var, bw, eps = bnp
    return _ops().bn_relu_bwd(g, keep, mean, var, bw, eps)


class _MaskScaleFn(torch.autograd.Function):
    """Identity in forward on the fused conv->BN->ReLU output; keeps the ReLU bit
    mask and in backward returns g * keep * s (one pass, ms_bn_relu_bwd).  A
    separate autograd node so the engine frees the incoming gradient before the
    dgrad allocates dX (two activation-sized buffers live, as unfused)."""

    @staticmethod
    def forward(ctx, y, mask, bn):
        # bn is None for the residual join: then only the ReLU mask is applied
        ctx.bn = None if bn is None else (bn.running_mean, bn.running_var, bn.weight,
                                          float(bn.eps))
        ctx.save_for_backward(mask)
        ctx.fmt = torch.channels_last if _is_channels_last(y) and not y.is_contiguous() \
            else torch.contiguous_format
        # y (the fused conv's fresh output, saved by nobody) is returned as itself and
        # marked dirty rather than as a view, so in-place consumers (ReLU(inplace=True),
        # add_, inplace dropout) stay legal as on the unfused layers
        ctx.mark_dirty(y)
        return y

    @staticmethod
    def backward(ctx, gy):
        (mask,) = ctx.saved_tensors
        mask = _need(mask, "mask", "conv_bn_relu dX")
        g = gy.contiguous(memory_format=ctx.fmt)
        if _is_meta(g):
            return torch.empty_like(g, memory_format=ctx.fmt), None, None
        if ctx.bn is None:
            return _ops().relu_bwd(g, mask), None, None
        mean, var, bw, eps = ctx.bn
        return _ops().bn_relu_bwd(g, mask, mean, var, bw, eps), None, None


def conv_bn_fusable(x: torch.Tensor, conv, bn) -> bool:
    """The fused launch applies: frozen eval-mode BN, plain conv (groups = dilation
    = 1, zeros padding), 16-bit activations on CUDA, K % 8 == 0."""
    if not _bn_frozen_eval(bn) or x.dim() != 4:
        return False
    if conv.groups != 1 or tuple(conv.dilation) != (1, 1) or conv.padding_mode != "zeros":
        return False
    if isinstance(conv.padding, str) or conv.out_channels % 8:
        return False
    if x.device.type == "meta":
        return x.dtype in (torch.bfloat16, torch.float16)
    return x.device.type == "cuda" and x.dtype in (torch.bfloat16, torch.float16) \
        and conv.weight.dtype == x.dtype and bn.running_mean.device == x.device


def _relu_keep_mask(y: torch.Tensor) -> torch.Tensor:
    # a ReLU folded into a fused call keeps its MemSave storage (bit mask); CPU
    # tensors raise inside relu() like every other entry point (no CPU path)
    return relu(y)


def fused_conv(x: torch.Tensor, conv, bn, relu_: bool, residual=None, tee: bool = False,
               in_mask=None, in_bn=None, raw: bool = False):
    """The general fused chain ``relu?(bn?(conv(x)) [+ residual])`` behind the
    wrappers below and the graph pass (nn.fuse_conv_bn_relu).  Returns
    ``(y, mask, alias)``:

    * ``tee``: alias is x itself for x's other consumer (else None); that
      consumer's gradient is summed into dX in the dgrad epilogue.
    * ``raw``: the ReLU's backward is NOT applied here; mask is its bit mask
      (else None) and the single consumer of y must be a fused conv that gets
      it as ``in_mask`` (with ``in_bn`` = this BN when the chain has one and no
      residual) and applies keep [* s] in its own dgrad epilogue.
    * ``in_mask`` / ``in_bn``: the producer's mask / BN for the above.

    One tcgen05 launch when the chain is fusable (frozen eval BN, 16-bit NHWC on
    CUDA); otherwise the layers in sequence, the producer's deferred ReLU
    backward applied first."""
    if in_mask is None:
        in_bn = None
    ok = conv_bn_fusable(x, conv, bn) if bn is not None else conv_relu_fusable(x, conv)
    if ok and residual is not None:
        # the epilogue reads the residual at full output indexing: no broadcasting
        oh, ow = _conv_out_hw(x.shape, conv.weight.shape, _pair(conv.stride), _pair(conv.padding))
        ok = residual.dtype == x.dtype and residual.device == x.device \
            and tuple(residual.shape) == (x.shape[0], conv.out_channels, oh, ow)
    # tee only a differentiable x: otherwise the alias would make x's other
    # consumer see requires_grad=True and run (and save for) a discarded dgrad
    tee_grad = tee and x.requires_grad
    if not ok:
        if in_mask is not None:
            x = _MaskScaleFn.apply(x, in_mask, in_bn)
        if tee_grad and _FALLBACK_TEE and conv_relu_fusable(x, conv):
            # the conv alone still runs tee'd: x's other gradient summed in its dgrad
            y, _, xt = _ConvBNFn.apply(x, conv.weight, conv.bias, None, conv.stride,
                                       conv.padding, None, False, True)
        else:
            xt = x if tee else None
            y = conv(x)
        if bn is not None and relu_ and bn_relu_fusable(y, bn) and (
                residual is None or (residual.shape == y.shape and residual.dtype == y.dtype)):
            # BN not absorbable (trainable affine): BN [-> + residual] -> ReLU in one pass
            return batch_norm_relu_eval(y, bn, residual), None, xt
        if bn is not None:
            y = bn(y)
        if residual is not None:
            y = add_relu(y, residual) if relu_ else y + residual
        elif relu_:
            y = _relu_keep_mask(y)
        return y, None, xt
    outs = _ConvBNFn.apply(x, conv.weight, conv.bias, residual, conv.stride, conv.padding, bn,
                           relu_, tee_grad, in_mask, in_bn)
    y, mask = outs[0], outs[1]
    if relu_ and mask is not None and not raw:
        # conv -> BN -> ReLU: g * keep * s; with a residual (BN scale folded into the
        # dgrad weight) or without a BN: g * keep
        y = _MaskScaleFn.apply(y, mask, bn if residual is None else None)
        mask = None
    alias = outs[2] if tee_grad else (x if tee else None)
    return y, (mask if raw else None), alias


def conv_bn_relu(x: torch.Tensor, conv, bn, with_relu: bool) -> torch.Tensor:
    """conv -> bn -> (relu) of the given modules: one fused launch when
    ``conv_bn_fusable`` holds, else the layers in sequence (BN in training mode
    or with trainable parameters, float32, ...)."""
    return fused_conv(x, conv, bn, with_relu)[0]


def conv_bn_relu_tee(x: torch.Tensor, conv, bn, with_relu: bool):
    """(conv_bn_relu(x, conv, bn, with_relu), x'): x' is x itself (a view, no
    copy) for x's other consumer, e.g. the identity or downsample branch of a
    ResNet block.  Its gradient is added to dX inside the dgrad epilogue, which
    replaces the engine's separate accumulation pass over the two gradients."""
    y, _, xt = fused_conv(x, conv, bn, with_relu, tee=True)
    return y, xt


# a tee'd conv runs through the fused kernel on the unfused (trainable-BN) path
# too, so the block input's second gradient is summed in the dgrad epilogue
# (residual-style addend prefetched ahead of the TMEM read) instead of by an
# autograd add; MS_FALLBACK_TEE=0 restores the plain module call
_FALLBACK_TEE = os.environ.get("MS_FALLBACK_TEE", "1") == "1"


def conv_relu_fusable(x: torch.Tensor, conv) -> bool:
    if x.dim() != 4 or conv.groups != 1 or tuple(conv.dilation) != (1, 1):
        return False
    if conv.padding_mode != "zeros" or isinstance(conv.padding, str) or conv.out_channels % 8:
        return False
    if x.device.type == "meta":
        return x.dtype in (torch.bfloat16, torch.float16)
    return x.device.type == "cuda" and x.dtype in (torch.bfloat16, torch.float16) \
        and conv.weight.dtype == x.dtype


def conv_relu(x: torch.Tensor, conv) -> torch.Tensor:
    """relu(conv(x)) with the ReLU (and its bit mask) in the conv epilogue (VGG);
    the two memsave layers in sequence when the fused launch does not apply."""
    return fused_conv(x, conv, None, True)[0]


def conv_bn_add_relu(x: torch.Tensor, conv, bn, residual: torch.Tensor) -> torch.Tensor:
    """relu(bn(conv(x)) + residual): the main branch and the join of a ResNet
    block in one launch (residual added in the conv epilogue) when
    ``conv_bn_fusable`` holds and the residual matches the output."""
    return fused_conv(x, conv, bn, True, residual)[0]


# =============================================================== fused residual add + ReLU
class _AddReLUFn(torch.autograd.Function):
    """relu(a + b) with the ReLU's bit mask (rules.py:98-101; the add saves
    nothing, rules.py:116-117); backward: one masked gradient for both operands."""

    @staticmethod
    def forward(ctx, a, b):
        out_rg = ctx.needs_input_grad[0] or ctx.needs_input_grad[1]
        n = a.numel()
        if _is_meta(a, b):
            ctx.save_for_backward(torch.empty((n + 7) // 8, dtype=torch.uint8, device="meta")
                                  if out_rg else None)
            ctx.fmt = torch.contiguous_format
            return a.new_empty(a.shape)
        _require_cuda("add_relu", a, b)
        fmt = _dense_format(a)
        if fmt is None or _dense_format(b) != fmt or a.dtype != b.dtype or a.shape != b.shape:
            raise RuntimeError("add_relu: operands must share shape, dtype and a dense layout")
        ctx.fmt = fmt
        _dtype_code(a)
        y, mask = _ops().add_relu_fwd(a, b, bool(out_rg))
        ctx.save_for_backward(_opt(mask, out_rg))
        return y

    @staticmethod
    def backward(ctx, gy):
        (mask,) = ctx.saved_tensors
        mask = _need(mask, "mask", "add_relu backward")
        g = gy.contiguous(memory_format=ctx.fmt)
        if _is_meta(g):
            dx = g.new_empty(g.shape)
            return (dx if ctx.needs_input_grad[0] else None,
                    dx if ctx.needs_input_grad[1] else None)
        dx = _ops().relu_bwd(g, mask)
        return (dx if ctx.needs_input_grad[0] else None,
                dx if ctx.needs_input_grad[1] else None)


def add_relu(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """relu(a + b) in one pass (the residual add of a ResNet block + its ReLU)."""
    fa, fb = _dense_format(a), _dense_format(b)
    if (a.device.type in ("cuda", "meta") and a.shape == b.shape and a.dtype == b.dtype
            and fa is not None and fa == fb):
        return _AddReLUFn.apply(a, b)
    return relu(a + b)
