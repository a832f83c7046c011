"""CPU oracle for the selective-save layers — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithm of the hot path
(``/root/reference/pkg/src/leantape``) so that the CUDA product path can be
checked against it.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it, and
there only as the checker or the timed CPU baseline — never as the product.
The product path (``paper_2404_12406_b200``) never imports this package and
fails loudly when its CUDA library is missing.

Parity pinning: the conv restatement and the storage-rule table are pinned
against golden vectors produced by importing the reference itself
(``oracle/gen_golden.py`` → ``tests/golden/*.npz``).  Linear and BatchNorm-eval
exist in the reference only as SPEC formulas; their
golden vectors come from the same formulas evaluated by torch-CPU float64 and
are therefore "pinned to the SPEC", not to reference code.
"""

from .conv import conv2d_fwd, conv2d_dx, conv2d_dw, conv_out_size  # noqa: F401
from .linear import linear_fwd, linear_dx, linear_dw, linear_db  # noqa: F401
from .batchnorm import bn_eval_fwd, bn_eval_dx, bn_eval_dw, bn_eval_db  # noqa: F401
from .pool import maxpool2d_fwd, maxpool2d_bwd, relu_fwd, relu_bwd  # noqa: F401
from .rules import Policy, storage_decision, linear_family  # noqa: F401
from .dropout import dropout_fwd, dropout_bwd, dropout_mask, uniforms  # noqa: F401
from .layernorm import layernorm_fwd, layernorm_bwd  # noqa: F401
from .gelu import gelu_fwd, gelu_bwd  # noqa: F401
from .conv_transpose import (conv_transpose2d_fwd, conv_transpose2d_dx,  # noqa: F401
                             conv_transpose2d_dw, conv_transpose2d_db)
from .tolerance import assert_close_fp32, assert_close_lowp, round_to  # noqa: F401
