"""Alias of :mod:`paper_2404_12406_b200.nn` under the upstream package name:
every MemSave layer, the converter and the fusion pass."""

from paper_2404_12406_b200.nn import (  # noqa: F401
    MemSaveBatchNorm2d,
    MemSaveConv2d,
    MemSaveConvTranspose2d,
    MemSaveDropout,
    MemSaveLayerNorm,
    MemSaveLinear,
    MemSaveMaxPool2d,
    MemSaveReLU,
    convert_to_memory_saving,
    fuse_conv_bn_relu,
    fuse_linear_dropout_add,
    fuse_linear_gelu,
)
from paper_2404_12406_b200.nn import __all__  # noqa: F401
