"""CPU port of the benchmark workloads on the reference algorithm — used ONLY
by bench.py's ``cpu_baseline`` leg and by ``bench.py --impl reference``.

The reference (leantape) is a CPU numpy/numba library; its conv kernels are
restated in oracle/conv.py (numpy_impl.py:12-51) and its Linear / BN-eval
VJPs in oracle/linear.py, oracle/batchnorm.py.  This module
strings them into the same network step the GPU arm runs (ResNet-18,
frozen weights, input-only gradient), in float32 — the dtype the reference
computes in — with numpy's BLAS threads on all host cores.  ReLU / MaxPool /
AvgPool are written inline (reference rules.py:98-109 kinds, not on the hot
path); MaxPool follows the reference's first-occurrence tie-break
(numpy_impl.py:54-70).
"""

from __future__ import annotations

import time

import numpy as np

import oracle

F32 = np.float32


def _bn_consts(sd, name, eps):
    w = sd[f"{name}.weight"].astype(np.float64)
    b = sd[f"{name}.bias"].astype(np.float64)
    m = sd[f"{name}.running_mean"].astype(np.float64)
    v = sd[f"{name}.running_var"].astype(np.float64)
    inv = 1.0 / np.sqrt(v + eps)
    scale = (w * inv).astype(F32)
    shift = (b - m * w * inv).astype(F32)
    return scale[None, :, None, None], shift[None, :, None, None]


def _maxpool_fwd(x, k=3, s=2, p=1):
    n, c, h, w = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)), constant_values=-np.inf)
    oh = (h + 2 * p - k) // s + 1
    ow = (w + 2 * p - k) // s + 1
    out = np.full((n, c, oh, ow), -np.inf, dtype=x.dtype)
    idx = np.zeros((n, c, oh, ow), dtype=np.int64)
    for i in range(k):
        for j in range(k):
            cand = xp[:, :, i:i + s * (oh - 1) + 1:s, j:j + s * (ow - 1) + 1:s]
            better = cand > out
            out = np.where(better, cand, out)
            idx = np.where(better, i * k + j, idx)
    return out, idx


def _maxpool_bwd(g, idx, h, w, k=3, s=2, p=1):
    n, c, oh, ow = g.shape
    dxp = np.zeros((n, c, h + 2 * p, w + 2 * p), dtype=g.dtype)
    for i in range(k):
        for j in range(k):
            sel = np.where(idx == i * k + j, g, 0)
            dxp[:, :, i:i + s * (oh - 1) + 1:s, j:j + s * (ow - 1) + 1:s] += sel
    return dxp[:, :, p:p + h, p:p + w]


class ResNet18InputGradCPU:
    """fwd + input-gradient bwd of torchvision ResNet-18 in eval mode, numpy f32."""

    def __init__(self, state_dict: dict, eps: float = 1e-5):
        self.sd = {k: v.detach().float().cpu().numpy() for k, v in state_dict.items()}
        self.eps = eps

    def _conv(self, x, name, s, p):
        return oracle.conv2d_fwd(x, self.sd[f"{name}.weight"], s, p, dtype=F32)

    def _conv_dx(self, g, name, s, p, h, w):
        return oracle.conv2d_dx(g, self.sd[f"{name}.weight"], s, p, h, w, dtype=F32)

    def step(self, x: np.ndarray, labels: np.ndarray) -> float:
        sd, eps = self.sd, self.eps
        tape = []
        # ---- forward
        h = self._conv(x, "conv1", 2, 3)
        sc, sf = _bn_consts(sd, "bn1", eps)
        h = h * sc + sf
        m0 = h > 0
        h = np.where(m0, h, 0).astype(F32)
        hp, pidx = _maxpool_fwd(h)
        pre_pool_hw = h.shape[2:]
        h = hp
        for li in range(1, 5):
            for bi in range(2):
                pre = f"layer{li}.{bi}"
                stride = 2 if (li > 1 and bi == 0) else 1
                inp = h
                a = self._conv(inp, f"{pre}.conv1", stride, 1)
                s1, f1 = _bn_consts(sd, f"{pre}.bn1", eps)
                a = a * s1 + f1
                ma = a > 0
                a = np.where(ma, a, 0).astype(F32)
                b = self._conv(a, f"{pre}.conv2", 1, 1)
                s2, f2 = _bn_consts(sd, f"{pre}.bn2", eps)
                b = b * s2 + f2
                if f"{pre}.downsample.0.weight" in sd:
                    idn = self._conv(inp, f"{pre}.downsample.0", stride, 0)
                    sd_, fd_ = _bn_consts(sd, f"{pre}.downsample.1", eps)
                    idn = idn * sd_ + fd_
                else:
                    idn = inp
                out = b + idn
                mo = out > 0
                h = np.where(mo, out, 0).astype(F32)
                tape.append((pre, stride, inp.shape, ma, mo, s1, s2))
        feat = h.mean(axis=(2, 3))
        logits = oracle.linear_fwd(feat, sd["fc.weight"], sd["fc.bias"]).astype(F32)
        # ---- loss (mean cross-entropy) and its gradient
        z = logits - logits.max(axis=1, keepdims=True)
        pz = np.exp(z)
        pz /= pz.sum(axis=1, keepdims=True)
        nb = x.shape[0]
        loss = float(-np.log(pz[np.arange(nb), labels]).mean())
        gl = pz
        gl[np.arange(nb), labels] -= 1.0
        gl = (gl / nb).astype(F32)
        # ---- backward (input gradient only: W frozen -> no dW products)
        gfeat = oracle.linear_dx(gl, sd["fc.weight"]).astype(F32)
        hw = h.shape[2] * h.shape[3]
        g = np.broadcast_to(gfeat[:, :, None, None] / hw, h.shape).astype(F32)
        for pre, stride, in_shape, ma, mo, s1, s2 in reversed(tape):
            g = np.where(mo, g, 0).astype(F32)
            gb = g * s2
            ga = self._conv_dx(gb, f"{pre}.conv2", 1, 1, ma.shape[2], ma.shape[3])
            ga = np.where(ma, ga, 0) * s1
            gin = self._conv_dx(ga, f"{pre}.conv1", stride, 1, in_shape[2], in_shape[3])
            if f"{pre}.downsample.0.weight" in sd:
                sd_, _ = _bn_consts(sd, f"{pre}.downsample.1", eps)
                gin = gin + self._conv_dx(g * sd_, f"{pre}.downsample.0", stride, 0, in_shape[2],
                                          in_shape[3])
            else:
                gin = gin + g
            g = gin.astype(F32)
        g = _maxpool_bwd(g, pidx, *pre_pool_hw)
        g = np.where(m0, g, 0) * _bn_consts(sd, "bn1", eps)[0]
        gx = self._conv_dx(g.astype(F32), "conv1", 2, 3, x.shape[2], x.shape[3])
        self.last_grad = gx
        return loss


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
