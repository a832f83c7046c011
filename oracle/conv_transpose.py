"""ConvTranspose2d (oracle) — TEST INFRASTRUCTURE ONLY.

SPEC.md forward_conv_transpose2d: "conv_transpose2d's forward equals conv2d's
input-VJP with the same kernel".  With weight [C_in][C_out][kh][kw] read as a
conv kernel [K = C_in][C = C_out][R][S], the three products are the
reference conv kernels (numpy_impl.py:12-51, restated in oracle/conv.py):
  y  = conv2d_dx(x, W)            (the conv "input" has C_out channels)
  dX = conv2d_fwd(g, W)
  dW = conv2d_dw(g, x)            (conv input g, conv output-gradient x)
  db = Σ g over N, H, W
"""

from __future__ import annotations

import numpy as np

from .conv import conv2d_dw, conv2d_dx, conv2d_fwd


def conv_transpose2d_fwd(x, w, b, stride, pad, output_padding=0):
    n, cin, h, wd = np.shape(x)
    kh, kw = np.shape(w)[2:]
    ho = (h - 1) * stride - 2 * pad + kh + output_padding
    wo = (wd - 1) * stride - 2 * pad + kw + output_padding
    y = conv2d_dx(x, w, stride, pad, ho, wo)
    if b is not None:
        y = y + np.asarray(b, dtype=np.float64).reshape(1, -1, 1, 1)
    return y


def conv_transpose2d_dx(g, w, stride, pad):
    return conv2d_fwd(g, w, stride, pad)


def conv_transpose2d_dw(x, g, stride, pad, kh, kw):
    return conv2d_dw(g, x, stride, pad, kh, kw)


def conv_transpose2d_db(g):
    return np.asarray(g, dtype=np.float64).sum(axis=(0, 2, 3))
