"""B200-native selective-save layers (arXiv 2404.12406, "Lowering PyTorch's
Memory Consumption for Selective Differentiation").

Public API (drop-in for ``memsave_torch``):
    paper_2404_12406_b200.nn.MemSaveLinear / MemSaveConv2d / MemSaveBatchNorm2d
    paper_2404_12406_b200.nn.convert_to_memory_saving
    paper_2404_12406_b200.functional.linear / conv2d / batch_norm_eval
    paper_2404_12406_b200.distributed.TrainableGradAllReduce
"""

from . import rules  # noqa: F401
from ._lib import LIB_PATH, launch_count, launch_stats, lib  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # lazy submodules so that `import paper_2404_12406_b200` stays cheap
    if name in ("nn", "functional", "distributed", "planner"):
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
