"""Direct 2-d cross-correlation: forward, input-VJP, weight-VJP (oracle).

Restates the reference's numpy backend
(/root/reference/pkg/src/leantape/kernels/numpy_impl.py:12-51): accumulate over
kernel offsets (no patch matrix), NCHW activations, OIHW weights, square int
stride/padding, no groups/dilation.  The reference's numba backend
(numba_impl.py:14-75) computes the same sums in a different order.

Differences from the reference, all deliberate and documented:
  * every entry point casts to float64 before accumulating (the numba conv2d_dw
    accumulates 2M terms sequentially in the input dtype, numba_impl.py:75,
    which is not accurate enough to be a float32 oracle — SURVEY.md §8(c));
  * rectangular stride/padding tuples are accepted as well as ints (torch's
    nn.Conv2d allows them; the reference is square-only).
"""

from __future__ import annotations

import numpy as np


def _pair(v):
    if isinstance(v, (tuple, list)):
        return int(v[0]), int(v[1])
    return int(v), int(v)


def conv_out_size(size: int, k: int, stride: int, padding: int) -> int:
    """OH = (H + 2p - kh) // s + 1 (numpy_impl.py:15-16)."""
    return (size + 2 * padding - k) // stride + 1


def conv2d_fwd(x, w, stride=1, padding=0, dtype=np.float64):
    """out[b,co,i,j] = sum_{ci,p,q} x[b,ci,i*s-pad+p, j*s-pad+q] * w[co,ci,p,q].

    Follows numpy_impl.py:12-24 (pad + one einsum per kernel offset).
    ``dtype`` is the accumulation dtype: float64 when checking; the CPU
    baseline passes float32, which is what the reference computes in.
    """
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    x = np.asarray(x, dtype=dtype)
    w = np.asarray(w, dtype=dtype)
    n, cin, h, wd = x.shape
    cout, _, kh, kw = w.shape
    oh = conv_out_size(h, kh, sh, ph)
    ow = conv_out_size(wd, kw, sw, pw)
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    out = np.zeros((n, cout, oh, ow), dtype=dtype)
    for i in range(kh):
        for j in range(kw):
            xs = xp[:, :, i:i + sh * (oh - 1) + 1:sh, j:j + sw * (ow - 1) + 1:sw]
            out += np.einsum("nchw,oc->nohw", xs, w[:, :, i, j], optimize=True)
    return out


def conv2d_dx(g, w, stride, padding, h, wd, dtype=np.float64):
    """Input-VJP as a scatter (transpose conv), numpy_impl.py:27-38.

    ``h, wd`` are explicit because stride > 1 makes the input size ambiguous.
    """
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    g = np.asarray(g, dtype=dtype)
    w = np.asarray(w, dtype=dtype)
    n, cout, oh, ow = g.shape
    _, cin, kh, kw = w.shape
    dxp = np.zeros((n, cin, h + 2 * ph + sh, wd + 2 * pw + sw), dtype=dtype)
    for i in range(kh):
        for j in range(kw):
            contrib = np.einsum("nohw,oc->nchw", g, w[:, :, i, j], optimize=True)
            dxp[:, :, i:i + sh * (oh - 1) + 1:sh, j:j + sw * (ow - 1) + 1:sw] += contrib
    return np.ascontiguousarray(dxp[:, :, ph:ph + h, pw:pw + wd])


def conv2d_dw(x, g, stride, padding, kh, kw, dtype=np.float64):
    """Weight-VJP, numpy_impl.py:41-51: dw[co,ci,p,q] = sum g * shifted x."""
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    x = np.asarray(x, dtype=dtype)
    g = np.asarray(g, dtype=dtype)
    n, cin, h, wd = x.shape
    _, cout, oh, ow = g.shape
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph + sh), (pw, pw + sw)))
    dw = np.zeros((cout, cin, kh, kw), dtype=dtype)
    for i in range(kh):
        for j in range(kw):
            xs = xp[:, :, i:i + sh * (oh - 1) + 1:sh, j:j + sw * (ow - 1) + 1:sw]
            dw[:, :, i, j] = np.einsum("nohw,nchw->oc", g, xs, optimize=True)
    return dw


def conv2d_db(g):
    """db = sum of G over N, H, W."""
    return np.asarray(g, dtype=np.float64).sum(axis=(0, 2, 3))
