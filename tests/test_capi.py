"""The C-ABI library loads and exports every symbol include/memsave_b200.h
declares (no compute calls — this runs without a GPU)."""

import ctypes
import os
import re

from paper_2404_12406_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "memsave_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"MS_API\s+[\w\s\*]+?\b(ms_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("ms_conv2d_fwd", "ms_conv2d_dx", "ms_conv2d_dw", "ms_linear_fwd", "ms_linear_dx",
              "ms_linear_dw", "ms_bn_eval_fwd", "ms_bn_eval_bwd", "ms_bias_grad"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_host_only_queries():
    L = _lib.lib()
    assert L.ms_version() >= 1
    assert L.ms_status_string(0) == b"MS_OK"
    assert L.ms_status_string(4) == b"MS_ERR_UNSUPPORTED"
    d = _lib.ConvDesc(256, 3, 224, 224, 64, 7, 7, 2, 2, 3, 3, _lib.MS_NHWC, _lib.MS_NHWC,
                      _lib.MS_BF16)
    assert L.ms_conv2d_out_h(ctypes.byref(d)) == 112
    assert L.ms_conv2d_out_w(ctypes.byref(d)) == 112
    # stem: 3 channels -> padded activation copy + repacked weight in the workspace
    assert L.ms_conv2d_workspace(ctypes.byref(d), _lib.MS_CONV_FWD) > 0
    assert L.ms_bn_eval_workspace(2, 64, 49, _lib.MS_NHWC) == 2 * 64 * 4


def test_invalid_descriptor_rejected_without_gpu():
    L = _lib.lib()
    d = _lib.ConvDesc(1, 0, 8, 8, 4, 3, 3, 1, 1, 1, 1, _lib.MS_NHWC, _lib.MS_NHWC, _lib.MS_BF16)
    st = L.ms_conv2d_fwd(ctypes.byref(d), None, None, None, None, None, 0, None)
    assert st == 1  # MS_ERR_SHAPE
    assert b"non-positive" in L.ms_last_error()
