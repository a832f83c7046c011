"""Storage-dependency table for the hot-path layer kinds (oracle).

Restates /root/reference/pkg/src/leantape/rules.py for the rows on the hot
path: linear (rules.py:64-66), conv2d / conv_transpose2d (rules.py:68-71),
batchnorm2d in eval mode (rules.py:84-87) and the shared ``_linear_family``
rule (rules.py:133-141), plus the first "next" rows: relu (rules.py:98-101)
and maxpool2d (rules.py:108-109), then dropout (rules.py:103-106) and layernorm
(rules.py:89-96).  Golden tables produced by importing the reference
(tests/golden/rules.json) pin this restatement.
"""

from __future__ import annotations

import enum


class Policy(enum.Enum):
    NAIVE = "naive"
    MEMSAVE = "memsave"


def linear_family(x_rg: bool, w_rg: bool):
    """rules.py:133-141 — the input VJP reads only W, the weight VJP only X,
    the bias VJP reads nothing."""
    saves = []
    if w_rg:
        saves.append(("x", "full"))
    if x_rg:
        saves.append(("w", "full"))
    return saves


def storage_decision(kind: str, policy: Policy, *, x_rg: bool, w_rg: bool,
                     out_rg: bool, bn_train: bool = False):
    if kind == "linear":
        return linear_family(x_rg, w_rg)
    if kind in ("conv2d", "conv_transpose2d"):
        if policy is Policy.MEMSAVE:
            return linear_family(x_rg, w_rg)
        return [("x", "full"), ("w", "full")] if out_rg else []
    if kind == "batchnorm2d":
        if bn_train:
            saves = []
            if x_rg or w_rg:
                saves += [("x", "full"), ("stats", "stats")]
            if x_rg:
                saves.append(("w", "full"))
            return saves
        if policy is Policy.MEMSAVE:
            return linear_family(x_rg, w_rg)
        return [("x", "full"), ("w", "full")] if out_rg else []
    if kind == "relu":  # rules.py:98-101
        if not out_rg:
            return []
        return [("mask", "bitmask")] if policy is Policy.MEMSAVE else [("y", "full")]
    if kind == "maxpool2d":  # rules.py:108-109
        return [("idx", "indexmap")] if out_rg else []
    if kind == "dropout":  # rules.py:103-106
        if not out_rg:
            return []
        return [("seed", "seed")] if policy is Policy.MEMSAVE else [("mask", "bytemask")]
    if kind == "layernorm":  # rules.py:89-96, identical under both policies
        saves = []
        if x_rg or w_rg:
            saves += [("x", "full"), ("stats", "stats")]
        if x_rg:
            saves.append(("w", "full"))
        return saves
    raise ValueError(f"no hot-path storage rule for op kind {kind!r}")
