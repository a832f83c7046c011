"""Fully-connected layer, forward and VJPs (oracle).

The reference has no code for this layer; it is specified at SPEC.md:241-249:
``Z = X·Wᵀ + b``; ``dX = G·W``; ``dW = Gᵀ·X``; ``db = Σ G``.  X has rank ≥ 2
with the last dim equal to in_features; leading dims are flattened.
"""

from __future__ import annotations

import numpy as np


# ``dtype``: float64 when checking; the CPU baseline passes float32, the dtype
# the reference computes in.


def _flat(a, dtype=np.float64):
    a = np.asarray(a, dtype=dtype)
    return a.reshape(-1, a.shape[-1])


def linear_fwd(x, w, b=None, dtype=np.float64):
    x = np.asarray(x, dtype=dtype)
    z = _flat(x, dtype) @ np.asarray(w, dtype=dtype).T
    if b is not None:
        z = z + np.asarray(b, dtype=dtype)
    return z.reshape(x.shape[:-1] + (z.shape[-1],))


def linear_dx(g, w, dtype=np.float64):
    g = np.asarray(g, dtype=dtype)
    dx = _flat(g, dtype) @ np.asarray(w, dtype=dtype)
    return dx.reshape(g.shape[:-1] + (dx.shape[-1],))


def linear_dw(x, g, dtype=np.float64):
    return _flat(g, dtype).T @ _flat(x, dtype)


def linear_db(g, dtype=np.float64):
    return _flat(g, dtype).sum(axis=0)
