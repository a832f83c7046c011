"""LayerNorm over the trailing dims (oracle) — TEST INFRASTRUCTURE ONLY.

Spec only in the reference (SPEC.md forward_layernorm; storage rule
rules.py:89-96): per row of D elements,
  mean = Σx/D,  var = Σ(x − mean)²/D (biased),  rstd = 1/√(var + ε)
  y  = (x − mean)·rstd·w + b
  dX = rstd·(g·w − mean_j(g·w) − x̂·mean_j(g·w·x̂)),  x̂ = (x − mean)·rstd
  dW = Σ_rows g·x̂,   db = Σ_rows g
"""

from __future__ import annotations

import numpy as np


def _rows(x, d):
    x = np.asarray(x, dtype=np.float64)
    return x.reshape(-1, d)


def layernorm_fwd(x, w, b, eps, d):
    xr = _rows(x, d)
    mean = xr.mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(((xr - mean) ** 2).mean(axis=1, keepdims=True) + eps)
    y = (xr - mean) * rstd
    if w is not None:
        y = y * np.asarray(w, dtype=np.float64).reshape(1, d)
    if b is not None:
        y = y + np.asarray(b, dtype=np.float64).reshape(1, d)
    return y.reshape(np.shape(x)), mean.ravel(), rstd.ravel()


def layernorm_bwd(g, x, w, eps, d):
    xr, gr = _rows(x, d), _rows(g, d)
    mean = xr.mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(((xr - mean) ** 2).mean(axis=1, keepdims=True) + eps)
    xh = (xr - mean) * rstd
    gw = gr * (np.asarray(w, dtype=np.float64).reshape(1, d) if w is not None else 1.0)
    dx = rstd * (gw - gw.mean(axis=1, keepdims=True) - xh * (gw * xh).mean(axis=1, keepdims=True))
    return dx.reshape(np.shape(x)), (gr * xh).sum(axis=0), gr.sum(axis=0)
