"""The PyTorch custom-op layer: ``torch.ops.memsave.*`` from
``libmemsave_torch.so`` (csrc/torch_ops.cpp, TORCH_LIBRARY(memsave)).

Every op is a thin C++ wrapper over one C-ABI entry point of
``libmemsave_b200.so``: it allocates the outputs from the caching allocator,
sets a device guard and launches on the current CUDA stream.  Each op also has
a Meta kernel (same allocations, no launch), so FakeTensor / torch.compile /
torch.export see the real output shapes, and CUDA-graph capture works because
nothing synchronises.  There is no CPU kernel: CPU tensors raise.
"""

from __future__ import annotations

import os
import threading

import torch

from . import _lib

TORCH_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmemsave_torch.so")

_lock = threading.Lock()
_loaded = False


def _load() -> None:
    global _loaded
    with _lock:
        if _loaded:
            return
        _lib.lib()  # the C ABI first (a clear error if it was not built)
        if not os.path.exists(TORCH_LIB_PATH):
            raise _lib.MemsaveLibraryError(
                f"{TORCH_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ "
                f"as g; g.build()'` (or `make -C paper_2404_12406_b200/csrc`). There is no CPU "
                f"fallback.")
        torch.ops.load_library(TORCH_LIB_PATH)
        _loaded = True


class _Overloads:
    """The ``.default`` overload of every op as an attribute: calling an
    OpOverload directly skips the packet's overload resolution on each call."""

    def __init__(self, ns):
        names = sorted({q.split("::", 1)[1].split(".")[0]
                        for q in torch._C._dispatch_get_all_op_names()
                        if q.startswith("memsave::")})
        for name in names:
            setattr(self, name, getattr(ns, name).default)


_OV = None


def ops():
    """The memsave ops (``torch.ops.memsave.<name>.default``), loading the op
    library on first use."""
    global _OV
    if _OV is None:
        if not _loaded:
            _load()
        _OV = _Overloads(torch.ops.memsave)
    return _OV
