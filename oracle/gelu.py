"""GELU (erf form) and its VJP (oracle) -- TEST INFRASTRUCTURE ONLY.

The reference has no GELU; the fused Linear -> GELU node
(``functional.linear_gelu``) is checked as the composition of the SPEC
Linear (oracle/linear.py) and the published definition that
``torch.nn.functional.gelu(approximate='none')`` implements:
``gelu(x) = x/2 * (1 + erf(x / sqrt 2))``,
``gelu'(x) = Phi(x) + x * phi(x)``.
"""

from __future__ import annotations

import math

import numpy as np

_erf = np.vectorize(math.erf, otypes=[np.float64])


def gelu_fwd(x):
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def gelu_bwd(g, x):
    x = np.asarray(x, dtype=np.float64)
    cdf = 0.5 * (1.0 + _erf(x / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return np.asarray(g, dtype=np.float64) * (cdf + x * pdf)
