"""Fully-connected layer, forward and VJPs (oracle).

The reference has no code for this layer; it is specified at SPEC.md:241-249:
``Z = X·Wᵀ + b``; ``dX = G·W``; ``dW = Gᵀ·X``; ``db = Σ G``.  X has rank ≥ 2
with the last dim equal to in_features; leading dims are flattened.
"""

from __future__ import annotations

import numpy as np


def _flat(a):
    a = np.asarray(a, dtype=np.float64)
    return a.reshape(-1, a.shape[-1])


def linear_fwd(x, w, b=None):
    x = np.asarray(x, dtype=np.float64)
    z = _flat(x) @ np.asarray(w, dtype=np.float64).T
    if b is not None:
        z = z + np.asarray(b, dtype=np.float64)
    return z.reshape(x.shape[:-1] + (z.shape[-1],))


def linear_dx(g, w):
    g = np.asarray(g, dtype=np.float64)
    dx = _flat(g) @ np.asarray(w, dtype=np.float64)
    return dx.reshape(g.shape[:-1] + (dx.shape[-1],))


def linear_dw(x, g):
    return _flat(g).T @ _flat(x)


def linear_db(g):
    return _flat(g).sum(axis=0)
