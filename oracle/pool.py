"""ReLU (masked) and MaxPool2d (index map) — oracle.

* maxpool2d_fwd / maxpool2d_bwd restate the reference's numpy backend
  (/root/reference/pkg/src/leantape/kernels/numpy_impl.py:54-78): offsets are
  scanned in row-major order and a strict ``>`` keeps the first occurrence.
  Extension (torch semantics): optional zero-based padding filled with -inf.
  Returns both the reference's flat index (row*W + col, numpy_impl.py:66) and
  the window-local offset r*kw + s the B200 kernels store in one byte.
* relu_fwd / relu_bwd follow SPEC.md forward_relu (Masked variant): y =
  max(x, 0), mask = (y > 0) with ties at 0 -> 0, dX = G ⊙ mask.
"""

from __future__ import annotations

import numpy as np


def maxpool2d_fwd(x, kh, kw, sh, sw, ph=0, pw=0):
    x = np.asarray(x, dtype=np.float64)
    n, c, h, wd = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)), constant_values=-np.inf)
    oh = (h + 2 * ph - kh) // sh + 1
    ow = (wd + 2 * pw - kw) // sw + 1
    out = np.full((n, c, oh, ow), -np.inf)
    local = np.zeros((n, c, oh, ow), dtype=np.int64)
    for i in range(kh):
        for j in range(kw):
            cand = xp[:, :, i:i + sh * (oh - 1) + 1:sh, j:j + sw * (ow - 1) + 1:sw]
            better = cand > out
            out = np.where(better, cand, out)
            local = np.where(better, i * kw + j, local)
    rows = np.arange(oh)[:, None] * sh - ph + local // kw
    cols = np.arange(ow)[None, :] * sw - pw + local % kw
    flat = rows * wd + cols
    return out, local, flat


def maxpool2d_bwd(g, flat, h, wd):
    """Scatter G to the argmax positions (numpy_impl.py:73-78)."""
    g = np.asarray(g, dtype=np.float64)
    n, c, _, _ = g.shape
    dx = np.zeros((n * c, h * wd))
    rows = np.arange(n * c)[:, None]
    np.add.at(dx, (rows, np.asarray(flat).reshape(n * c, -1)), g.reshape(n * c, -1))
    return dx.reshape(n, c, h, wd)


def relu_fwd(x):
    x = np.asarray(x, dtype=np.float64)
    mask = x > 0
    return np.where(mask, x, 0.0), mask


def relu_bwd(g, mask):
    return np.where(mask, np.asarray(g, dtype=np.float64), 0.0)
