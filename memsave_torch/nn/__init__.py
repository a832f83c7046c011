"""Alias of :mod:`paper_2404_12406_b200.nn` under the upstream package name."""

from paper_2404_12406_b200.nn import (  # noqa: F401
    MemSaveBatchNorm2d,
    MemSaveConv2d,
    MemSaveLinear,
    MemSaveMaxPool2d,
    MemSaveReLU,
    convert_to_memory_saving,
)

__all__ = ["MemSaveLinear", "MemSaveConv2d", "MemSaveBatchNorm2d", "MemSaveReLU",
           "MemSaveMaxPool2d", "convert_to_memory_saving"]
