"""Import alias so code written against ``memsave_torch`` runs unchanged:
``import memsave_torch.nn`` resolves to :mod:`paper_2404_12406_b200.nn`."""

from paper_2404_12406_b200 import __version__  # noqa: F401
from . import nn  # noqa: F401
