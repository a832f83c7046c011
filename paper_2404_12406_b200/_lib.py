"""ctypes binding of the C-ABI library ``libmemsave_b200.so`` (include/memsave_b200.h).

The library is built in-tree (``__graft_entry__.build()`` or ``make -C
paper_2404_12406_b200/csrc``).  There is no CPU fallback anywhere in this
package: if the library is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmemsave_b200.so")

MS_F32, MS_BF16, MS_F16 = 0, 1, 2
MS_NCHW, MS_NHWC = 0, 1
MS_CONV_FWD, MS_CONV_DX, MS_CONV_DW = 0, 1, 2
MS_RNG_PHILOX4X32, MS_RNG_PHILOX4X64_REF = 0, 1

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_c_sz = ctypes.c_size_t
_vp = ctypes.c_void_p


class ConvDesc(ctypes.Structure):
    """ms_conv_desc (include/memsave_b200.h)."""

    _fields_ = [("n", _c_i64), ("c", _c_i64), ("h", _c_i64), ("w", _c_i64),
                ("k", _c_i64), ("r", _c_i64), ("s", _c_i64),
                ("stride_h", _c_i32), ("stride_w", _c_i32),
                ("pad_h", _c_i32), ("pad_w", _c_i32),
                ("layout", _c_i32), ("wlayout", _c_i32), ("dtype", _c_i32)]


class PoolDesc(ctypes.Structure):
    """ms_pool_desc (include/memsave_b200.h)."""

    _fields_ = [("n", _c_i64), ("c", _c_i64), ("h", _c_i64), ("w", _c_i64),
                ("kh", _c_i32), ("kw", _c_i32), ("stride_h", _c_i32), ("stride_w", _c_i32),
                ("pad_h", _c_i32), ("pad_w", _c_i32), ("layout", _c_i32), ("dtype", _c_i32)]


# (name, restype, argtypes) for every symbol the header declares
SIGNATURES = {
    "ms_conv2d_out_h": (_c_i64, [ctypes.POINTER(ConvDesc)]),
    "ms_conv2d_out_w": (_c_i64, [ctypes.POINTER(ConvDesc)]),
    "ms_conv2d_workspace": (_c_sz, [ctypes.POINTER(ConvDesc), _c_i32]),
    "ms_conv2d_fwd": (_c_i32, [ctypes.POINTER(ConvDesc), _vp, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_conv2d_dx": (_c_i32, [ctypes.POINTER(ConvDesc), _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_conv2d_dw": (_c_i32, [ctypes.POINTER(ConvDesc), _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_conv2d_db": (_c_i32, [ctypes.POINTER(ConvDesc), _vp, _vp, _vp, _c_sz, _vp]),
    "ms_linear_workspace": (_c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32]),
    "ms_linear_fwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_linear_gelu_fwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _c_sz, _vp]),
    "ms_linear_dropout_add_fwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _vp,
                                           ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                                           _c_i32, _vp, _vp, _c_sz, _vp]),
    "ms_gelu_fwd": (_c_i32, [_c_i64, _c_i32, _vp, _vp, _vp]),
    "ms_gelu_bwd": (_c_i32, [_c_i64, _c_i32, _vp, _vp, _vp, _vp]),
    "ms_linear_dx": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_linear_dw": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_bias_grad_workspace": (_c_sz, [_c_i64, _c_i64, _c_i32]),
    "ms_bias_grad": (_c_i32, [_c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_bn_eval_workspace": (_c_sz, [_c_i64, _c_i64, _c_i64, _c_i32]),
    "ms_bn_eval_fwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp,
                                _vp, _vp, ctypes.c_double, _vp, _vp, _c_sz, _vp]),
    "ms_bn_eval_bwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp,
                                _vp, _vp, ctypes.c_double, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_relu_fwd": (_c_i32, [_c_i64, _c_i32, _vp, _vp, _vp, _vp]),
    "ms_relu_bwd": (_c_i32, [_c_i64, _c_i32, _vp, _vp, _vp, _vp]),
    "ms_add_relu_fwd": (_c_i32, [_c_i64, _c_i32, _vp, _vp, _vp, _vp, _vp]),
    "ms_conv2d_bn_workspace": (_c_sz, [ctypes.POINTER(ConvDesc)]),
    "ms_conv2d_bn_fwd": (_c_i32, [ctypes.POINTER(ConvDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _c_i32, ctypes.c_double, _vp, _c_i32, _vp, _vp, _vp, _c_sz,
                                  _vp]),
    "ms_conv2d_bn_dx": (_c_i32, [ctypes.POINTER(ConvDesc), _vp, _vp, _vp, _vp, _c_i32,
                                 ctypes.c_double, _vp, _vp, _vp, _vp, _c_i32, ctypes.c_double,
                                 _vp, _vp, _c_sz, _vp]),
    "ms_bn_eval_relu_fwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _vp, _vp, _vp, _vp,
                                     _vp, ctypes.c_double, _vp, _vp, _vp]),
    "ms_bn_eval_relu_bwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _vp, _vp, _vp, _vp,
                                     _vp, _vp, ctypes.c_double, _vp, _vp, _vp, _vp, _c_sz, _vp]),
    "ms_bn_eval_add_relu_fwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _vp, _vp, _vp,
                                         _vp, _vp, _vp, ctypes.c_double, _vp, _vp, _vp]),
    "ms_bn_eval_add_relu_bwd": (_c_i32, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _vp, _vp, _vp,
                                         _vp, _vp, _vp, ctypes.c_double, _vp, _vp, _vp, _vp,
                                         _vp, _c_sz, _vp]),
    "ms_bn_relu_bwd": (_c_i32, [_c_i64, _c_i64, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp,
                                ctypes.c_double, _vp, _vp]),
    "ms_maxpool2d_out_h": (_c_i64, [ctypes.POINTER(PoolDesc)]),
    "ms_maxpool2d_out_w": (_c_i64, [ctypes.POINTER(PoolDesc)]),
    "ms_maxpool2d_fwd": (_c_i32, [ctypes.POINTER(PoolDesc), _vp, _vp, _vp, _vp]),
    "ms_maxpool2d_bwd": (_c_i32, [ctypes.POINTER(PoolDesc), _vp, _vp, _vp, _vp]),
    "ms_maxpool2d_relu_bwd": (_c_i32, [ctypes.POINTER(PoolDesc), _vp, _vp, _vp, _vp, _vp, _c_i32,
                                       ctypes.c_double, _vp, _vp]),
    "ms_conv_transpose2d_fwd": (_c_i32, [ctypes.POINTER(ConvDesc), _vp, _vp, _vp, _vp, _vp, _c_sz,
                                         _vp]),
    "ms_dropout_fwd": (_c_i32, [_c_i64, _c_i32, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64,
                                ctypes.c_double, _c_i32, _vp, _vp]),
    "ms_dropout_bwd": (_c_i32, [_c_i64, _c_i32, _vp, _vp, ctypes.c_uint64, ctypes.c_uint64,
                                ctypes.c_double, _c_i32, _vp]),
    "ms_layernorm_workspace": (_c_sz, [_c_i64, _c_i64, _c_i32]),
    "ms_layernorm_fwd": (_c_i32, [_c_i64, _c_i64, _c_i32, _vp, _vp, _vp, ctypes.c_double, _vp,
                                  _vp, _vp, _vp]),
    "ms_layernorm_bwd": (_c_i32, [_c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _c_sz, _vp]),
    "ms_status_string": (ctypes.c_char_p, [_c_i32]),
    "ms_last_error": (ctypes.c_char_p, []),
    "ms_version": (_c_i32, []),
    "ms_launch_count": (_c_i64, []),
    "ms_launch_stats": (None, [ctypes.POINTER(_c_i64)]),
    "ms_set_device_bound": (None, [_c_i32]),
}

_lock = threading.Lock()
_lib = None


class MemsaveLibraryError(RuntimeError):
    pass


def lib():
    """Load (once) and return the CDLL; raises if the library was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise MemsaveLibraryError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (or `make -C paper_2404_12406_b200/csrc`). There is no CPU fallback.")
            h = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        L = lib()
        msg = L.ms_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed: {L.ms_status_string(status).decode()}: {msg}")


def launch_count() -> int:
    return int(lib().ms_launch_count())


FAMILIES = ("umma", "simt", "bn", "misc")


def launch_stats() -> dict:
    """Kernel launches since load, by family (tcgen05 GEMM, SIMT, BN, misc)."""
    buf = (_c_i64 * 4)()
    lib().ms_launch_stats(buf)
    return dict(zip(FAMILIES, (int(v) for v in buf)))
