"""Forward-time storage decision of the differentiability-agnostic layers.

Product-side statement of the reference rule table for the hot-path kinds
(/root/reference/pkg/src/leantape/rules.py:57-141, MEMSAVE policy):

  * linear, conv2d, conv_transpose2d, batchnorm2d (eval): the "linear family"
    (rules.py:133-141) — keep the layer input X iff the weight needs a
    gradient, keep the weight W iff the input needs a gradient; the bias VJP
    reads nothing.

The autograd functions in :mod:`.functional` call :func:`saved_roles` with
``ctx.needs_input_grad`` and pass exactly those tensors to
``ctx.save_for_backward``; the tests compare the result with the reference
table (tests/golden/rules.json, generated from the reference itself).
"""

from __future__ import annotations

# Kinds this package swaps (the hot-path subset of rules.CONVERTIBLE_KINDS,
# rules.py:51-52).
CONVERTIBLE_KINDS = ("linear", "conv2d", "batchnorm2d")


class MissingSavedValue(RuntimeError):
    """A backward product asked for a value the storage rule did not keep.

    Mirrors leantape.errors.MissingSavedValue (errors.py:20-25): firing means a
    storage rule is wrong; it must never happen for a correctly configured run.
    """


def saved_roles(x_rg: bool, w_rg: bool) -> tuple[str, ...]:
    """Roles kept for backward by a linear-family layer (rules.py:133-141)."""
    roles = []
    if w_rg:
        roles.append("x")
    if x_rg:
        roles.append("w")
    return tuple(roles)
