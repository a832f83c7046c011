"""Tolerance definitions used by every parity test.

* float32: compare against the float64 oracle; norm-wise relative error ≤ 1e-5
  AND elementwise |a − r| ≤ 1e-5·|r| + 1e-5·max|r|.  (Pure elementwise rtol 1e-5
  fails 0.5–10 % of elements for *any* float32 implementation.)
* bf16 / fp16: the oracle is evaluated in float64 on the same quantised inputs
  and rounded to the output dtype; require ≤ ``ulps`` output ulps elementwise
  (relative to max(|r|, atol_floor)) and norm-wise relative error ≤ 1e-3.
"""

from __future__ import annotations

import numpy as np

_MANT = {"bf16": 8, "fp16": 11, "f32": 24}


def round_to(a, dtype: str):
    """Round float64 values to bf16/fp16/f32 (round-to-nearest-even)."""
    a = np.asarray(a, dtype=np.float64)
    if dtype == "f32":
        return a.astype(np.float32).astype(np.float64)
    if dtype == "fp16":
        return a.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        f = a.astype(np.float32)
        u = f.view(np.uint32).astype(np.uint64)
        lsb = (u >> 16) & 1
        u = (u + 0x7FFF + lsb) & 0xFFFF0000
        return u.astype(np.uint32).view(np.float32).astype(np.float64)
    raise ValueError(dtype)


def norm_rel(a, r):
    a = np.asarray(a, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    den = np.linalg.norm(r.ravel())
    num = np.linalg.norm((a - r).ravel())
    return num / den if den > 0 else num


def assert_close_fp32(a, r, rtol=1e-5, what=""):
    a = np.asarray(a, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    assert a.shape == r.shape, (what, a.shape, r.shape)
    nr = norm_rel(a, r)
    assert nr <= rtol, f"{what}: norm-wise rel err {nr:.3e} > {rtol}"
    scale = float(np.max(np.abs(r))) if r.size else 0.0
    bad = np.abs(a - r) > rtol * np.abs(r) + rtol * scale
    assert not bad.any(), (f"{what}: {int(bad.sum())}/{bad.size} elements outside "
                           f"rtol={rtol} (max abs err {np.max(np.abs(a - r)):.3e})")


def assert_close_lowp(a, r64, dtype="bf16", ulps=2.0, norm_tol=1e-3, what="",
                      scale_floor_frac=1e-2):
    """``r64`` is the float64 oracle on the quantised inputs (unrounded).

    Elementwise bound: |a − round(r)| ≤ ulps · ulp(max(|r|, floor)), with
    floor = scale_floor_frac · max|r| so that catastrophic-cancellation outputs
    (|r| ≪ the terms summed) are judged against the magnitude of the terms.
    """
    a = np.asarray(a, dtype=np.float64)
    r64 = np.asarray(r64, dtype=np.float64)
    assert a.shape == r64.shape, (what, a.shape, r64.shape)
    rr = round_to(r64, dtype)
    nr = norm_rel(a, rr)
    assert nr <= norm_tol, f"{what}: norm-wise rel err {nr:.3e} > {norm_tol}"
    mag = np.maximum(np.abs(r64), scale_floor_frac * (np.max(np.abs(r64)) if r64.size else 0))
    ulp = np.exp2(np.floor(np.log2(np.maximum(mag, 1e-300))) - (_MANT[dtype] - 1))
    bad = np.abs(a - rr) > ulps * ulp
    assert not bad.any(), (f"{what}: {int(bad.sum())}/{bad.size} elements beyond {ulps} "
                           f"{dtype} ulps (max abs err {np.max(np.abs(a - rr)):.3e})")
