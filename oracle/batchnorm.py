"""BatchNorm2d in eval mode, forward and VJPs (oracle).

Spec only in the reference (running stats are module state
per SPEC.md:209-212 and :343):
  y  = W (x − μ̂)/√(σ̂² + ε) + b
  dX = G ⊙ W/√(σ̂² + ε)
  dW = Σ G ⊙ X̂ ,   X̂ = (x − μ̂)/√(σ̂² + ε)
  db = Σ G
Reductions run over N, H, W for each channel (axis 1 of NCHW).
"""

from __future__ import annotations

import numpy as np


def _c(v, x):
    return np.asarray(v, dtype=np.float64).reshape((1, -1) + (1,) * (x.ndim - 2))


def _invstd(var, eps):
    return 1.0 / np.sqrt(np.asarray(var, dtype=np.float64) + eps)


def bn_eval_fwd(x, mean, var, weight, bias, eps):
    x = np.asarray(x, dtype=np.float64)
    inv = _invstd(var, eps)
    w = np.ones_like(inv) if weight is None else np.asarray(weight, np.float64)
    b = np.zeros_like(inv) if bias is None else np.asarray(bias, np.float64)
    return (x - _c(mean, x)) * _c(inv * w, x) + _c(b, x)


def bn_eval_dx(g, var, weight, eps):
    g = np.asarray(g, dtype=np.float64)
    inv = _invstd(var, eps)
    w = np.ones_like(inv) if weight is None else np.asarray(weight, np.float64)
    return g * _c(w * inv, g)


def bn_eval_dw(g, x, mean, var, eps):
    g = np.asarray(g, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    xhat = (x - _c(mean, x)) * _c(_invstd(var, eps), x)
    axes = (0,) + tuple(range(2, x.ndim))
    return (g * xhat).sum(axis=axes)


def bn_eval_db(g):
    g = np.asarray(g, dtype=np.float64)
    return g.sum(axis=(0,) + tuple(range(2, g.ndim)))
