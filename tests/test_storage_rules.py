"""Saved-set identity (acceptance criterion 2).

For every hot-path layer and every (x_rg, w_rg, b_rg) combination the tensors
the autograd function hands to ``save_for_backward`` must equal the reference
rule table (tests/golden/rules.json, generated from leantape.rules).  Runs on
the ``meta`` device: shapes only, no arithmetic, no GPU.
"""

import itertools

import pytest
import torch

from paper_2404_12406_b200 import functional as MF
from paper_2404_12406_b200.rules import MissingSavedValue, saved_roles

FLAGS = list(itertools.product([False, True], repeat=3))


def _golden_saves(rules_golden, kind, x_rg, w_rg, b_rg, policy="memsave"):
    for row in rules_golden:
        if (row["kind"], row["policy"], row["x_rg"], row["w_rg"], row["b_rg"],
                row["bn_train"]) == (kind, policy, x_rg, w_rg, b_rg, False):
            return sorted(r for r, _k in row["saves"])
    raise KeyError(kind)


def _run(fn, tensors, roles_by_shape):
    packed = []

    def pack(t):
        packed.append(tuple(t.shape))
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = fn(*tensors)
    roles = sorted(roles_by_shape[s] for s in packed)
    return out, roles


def _make(shape, rg):
    return torch.empty(shape, device="meta").requires_grad_(rg)


@pytest.mark.parametrize("x_rg,w_rg,b_rg", FLAGS)
def test_linear_saved_set(rules_golden, x_rg, w_rg, b_rg):
    x, w, b = _make((6, 5, 7), x_rg), _make((3, 7), w_rg), _make((3,), b_rg)
    out, roles = _run(MF.linear, (x, w, b), {(6, 5, 7): "x", (3, 7): "w"})
    assert roles == _golden_saves(rules_golden, "linear", x_rg, w_rg, b_rg)
    assert out.shape == (6, 5, 3)
    if out.requires_grad:
        out.sum().backward()  # sufficiency: no MissingSavedValue
        assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg
        assert (b.grad is not None) == b_rg


@pytest.mark.parametrize("x_rg,w_rg,b_rg", FLAGS)
def test_conv2d_saved_set(rules_golden, x_rg, w_rg, b_rg):
    x, w, b = _make((2, 4, 9, 9), x_rg), _make((6, 4, 3, 3), w_rg), _make((6,), b_rg)
    out, roles = _run(lambda *t: MF.conv2d(*t, stride=2, padding=1), (x, w, b),
                      {(2, 4, 9, 9): "x", (6, 4, 3, 3): "w"})
    assert roles == _golden_saves(rules_golden, "conv2d", x_rg, w_rg, b_rg)
    assert out.shape == (2, 6, 5, 5)
    if out.requires_grad:
        out.sum().backward()
        assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg


@pytest.mark.parametrize("x_rg,w_rg,b_rg", FLAGS)
def test_batchnorm2d_eval_saved_set(rules_golden, x_rg, w_rg, b_rg):
    x, w, b = _make((2, 5, 4, 3), x_rg), _make((5,), w_rg), _make((5,), b_rg)
    rm, rv = torch.empty(5, device="meta"), torch.empty(5, device="meta")
    out, roles = _run(lambda x_, w_, b_: MF.batch_norm_eval(x_, rm, rv, w_, b_, 1e-5), (x, w, b),
                      {(2, 5, 4, 3): "x", (5,): "w"})
    assert roles == _golden_saves(rules_golden, "batchnorm2d", x_rg, w_rg, b_rg)
    if out.requires_grad:
        out.sum().backward()
        assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg


def test_bn_eval_input_scenario_saves_nothing_of_numel_size(rules_golden):
    # Eval, x diff, W frozen: nothing sized O(numel) is saved
    x = _make((2, 5, 4, 3), True)
    w, b = _make((5,), False), _make((5,), False)
    rm, rv = torch.empty(5, device="meta"), torch.empty(5, device="meta")
    _out, roles = _run(lambda: MF.batch_norm_eval(x, rm, rv, w, b), (), {(5,): "w",
                                                                          (2, 5, 4, 3): "x"})
    assert "x" not in roles


def test_saved_roles_is_the_linear_family():
    assert saved_roles(False, False) == ()
    assert saved_roles(True, False) == ("w",)
    assert saved_roles(False, True) == ("x",)
    assert saved_roles(True, True) == ("x", "w")


def test_missing_saved_value_fires():
    # The tripwire of errors.py:20-25: backward asking for an unsaved value raises.
    from paper_2404_12406_b200.functional import _need
    with pytest.raises(MissingSavedValue):
        _need(None, "x", "conv2d dW")


@pytest.mark.parametrize("kind", ["conv2d", "batchnorm2d"])
def test_stock_torch_matches_naive_row(rules_golden, kind):
    """Stock torch (CPU) is the reference's NAIVE policy for conv / BN-eval in the
    Input scenario: X and W are saved although W is frozen (Fig. 2 of the paper)."""
    x = torch.randn(2, 4, 6, 6, requires_grad=True)
    packed = []

    def pack(t):
        packed.append(tuple(t.shape))
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        if kind == "conv2d":
            w = torch.randn(3, 4, 3, 3)
            torch.nn.functional.conv2d(x, w, padding=1)
        else:
            torch.nn.functional.batch_norm(x, torch.zeros(4), torch.ones(4), torch.ones(4),
                                           torch.zeros(4), training=False)
    naive = _golden_saves(rules_golden, kind, True, False, False, policy="naive")
    assert naive == ["w", "x"]
    assert (2, 4, 6, 6) in packed  # stock keeps X; MemSave does not


@pytest.mark.parametrize("x_rg", [False, True])
def test_relu_saved_set_is_a_bitmask(rules_golden, x_rg):
    x = _make((2, 5, 4, 3), x_rg)
    packed = []

    def pack(t):
        packed.append((tuple(t.shape), t.dtype))
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = MF.relu(x)
    exp = _golden_saves(rules_golden, "relu", x_rg, False, False)
    assert exp == (["mask"] if x_rg else [])
    if x_rg:
        # one bit per element, not a copy of the output (saved.py:53-71)
        assert packed == [(((2 * 5 * 4 * 3 + 7) // 8,), torch.uint8)]
        out.sum().backward()
    else:
        assert packed == []


@pytest.mark.parametrize("x_rg", [False, True])
def test_maxpool_saved_set_is_an_index_map(rules_golden, x_rg):
    x = _make((2, 5, 9, 9), x_rg)
    packed = []

    def pack(t):
        packed.append((tuple(t.shape), t.dtype))
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = MF.max_pool2d(x, 3, 2, 1)
    exp = _golden_saves(rules_golden, "maxpool2d", x_rg, False, False)
    assert exp == (["idx"] if x_rg else [])
    assert out.shape == (2, 5, 5, 5)
    if x_rg:
        assert packed == [((2, 5, 5, 5), torch.uint8)]  # 1 byte per output element
        out.sum().backward()
    else:
        assert packed == []


# =============================================================== §8(f) rows
@pytest.mark.parametrize("x_rg", [False, True])
def test_dropout_saved_set_is_a_16_byte_key(rules_golden, x_rg):
    x = _make((4, 6, 10), x_rg)
    packed = []

    def pack(t):
        packed.append((tuple(t.shape), t.dtype, t.numel() * t.element_size()))
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = MF.dropout(x, 0.3, True, seed=5, stream=MF.DROPOUT_STREAM_BASE + 2)
    exp = _golden_saves(rules_golden, "dropout", x_rg, False, False)
    assert exp == (["seed"] if x_rg else [])
    if x_rg:
        # RngSeed: <= 16 bytes regardless of the tensor size (saved.py:91-108)
        assert packed == [((2,), torch.int64, 16)]
        out.sum().backward()
        assert x.grad.shape == x.shape
    else:
        assert packed == []


def test_dropout_eval_and_p0_are_identity():
    x = _make((3, 4), True)
    assert MF.dropout(x, 0.5, training=False) is x
    assert MF.dropout(x, 0.0, training=True) is x
    with pytest.raises(ValueError):
        MF.dropout(x, 1.0)


@pytest.mark.parametrize("x_rg,w_rg,b_rg", FLAGS)
def test_layernorm_saved_set(rules_golden, x_rg, w_rg, b_rg):
    x, w, b = _make((3, 5, 8), x_rg), _make((8,), w_rg), _make((8,), b_rg)
    packed = []

    def pack(t):
        packed.append((tuple(t.shape), t.dtype))
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = MF.layer_norm(x, (8,), w, b, 1e-5)
    role = {((3, 5, 8), torch.float32): "x", ((8,), torch.float32): "w",
            ((15,), torch.float32): "stats"}
    roles = sorted(set(role[p] for p in packed))
    assert roles == sorted(set(_golden_saves(rules_golden, "layernorm", x_rg, w_rg, b_rg)))
    if "stats" in roles:
        assert sum(1 for p in packed if role[p] == "stats") == 2  # mean and rstd per row
    if out.requires_grad:
        out.sum().backward()
        assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg
        assert (b.grad is not None) == b_rg


@pytest.mark.parametrize("x_rg,w_rg,b_rg", FLAGS)
def test_conv_transpose2d_saved_set(rules_golden, x_rg, w_rg, b_rg):
    x, w, b = _make((2, 4, 5, 5), x_rg), _make((4, 6, 3, 3), w_rg), _make((6,), b_rg)
    out, roles = _run(lambda *t: MF.conv_transpose2d(*t, stride=2, padding=1), (x, w, b),
                      {(2, 4, 5, 5): "x", (4, 6, 3, 3): "w"})
    assert roles == _golden_saves(rules_golden, "conv_transpose2d", x_rg, w_rg, b_rg)
    assert out.shape == (2, 6, 9, 9)
    if out.requires_grad:
        out.sum().backward()
        assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg
        assert (b.grad is not None) == b_rg


@pytest.mark.parametrize("x_rg,w_rg", [(True, False), (False, True), (True, True)])
def test_linear_without_bias_backward_on_meta(x_rg, w_rg):
    """memsave::linear with bias=None: the C++ autograd node has two inputs and
    returns only the requested gradients (Llama-style bias-free projections)."""
    x = torch.empty(4, 6, 7, device="meta").requires_grad_(x_rg)
    w = torch.empty(3, 7, device="meta").requires_grad_(w_rg)
    y = MF.linear(x, w, None)
    y.sum().backward()
    assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg
    if x_rg:
        assert x.grad.shape == x.shape
    if w_rg:
        assert w.grad.shape == w.shape


@pytest.mark.parametrize("x_rg,w_rg,b_rg", FLAGS)
def test_linear_gelu_saved_set(rules_golden, x_rg, w_rg, b_rg):
    """The fused Linear -> GELU node saves the Linear's rule set plus the GELU's
    input (the pre-activation, its VJP's only need), and nothing else."""
    x, w, b = _make((6, 5, 7), x_rg), _make((3, 7), w_rg), _make((3,), b_rg)
    out, roles = _run(MF.linear_gelu, (x, w, b), {(6, 5, 7): "x", (3, 7): "w", (6, 5, 3): "pre"})
    want = _golden_saves(rules_golden, "linear", x_rg, w_rg, b_rg)
    if x_rg or w_rg or b_rg:
        want = sorted(want + ["pre"])
    assert roles == want
    assert out.shape == (6, 5, 3)
    if out.requires_grad:
        out.sum().backward()
        assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg
        assert (b.grad is not None) == b_rg


@pytest.mark.parametrize("x_rg,w_rg,b_rg", FLAGS)
@pytest.mark.parametrize("r_rg", [False, True])
def test_linear_dropout_add_saved_set(rules_golden, x_rg, w_rg, b_rg, r_rg):
    """Linear -> dropout -> + residual as one node saves exactly the Linear's
    rule set: the dropout keeps its 16-byte key as node data, the add nothing."""
    x, w, b = _make((6, 5, 7), x_rg), _make((3, 7), w_rg), _make((3,), b_rg)
    r = _make((6, 5, 3), r_rg)
    out, roles = _run(lambda *t: MF.linear_dropout_add(*t, p=0.1, seed=7), (x, w, b, r),
                      {(6, 5, 7): "x", (3, 7): "w"})
    assert roles == _golden_saves(rules_golden, "linear", x_rg, w_rg, b_rg)
    assert out.shape == (6, 5, 3)
    if out.requires_grad:
        out.sum().backward()
        assert (x.grad is not None) == x_rg and (w.grad is not None) == w_rg
        assert (b.grad is not None) == b_rg and (r.grad is not None) == r_rg
