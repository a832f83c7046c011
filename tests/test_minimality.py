"""Minimality of the saved set (the reference instruments it with
``SavedValue.was_read``, saved.py:22-28): every tensor a MemSave layer keeps for
backward is read by an executed VJP, for every requires_grad combination.

Our instrument is the torch equivalent of ``was_read``: a
``saved_tensors_hooks`` pack/unpack pair that records every value the layer
saves and marks it when backward unpacks it.  On top, each full tensor kept is
checked against the VJP that consumes it (x only for a requested dW, W only for
a requested dX, reference rules.py:133-141).  Runs on the meta device."""

import itertools

import pytest
import torch
from torch import nn

import paper_2404_12406_b200.nn as pnn
from paper_2404_12406_b200 import functional as MF

BF = torch.bfloat16


class _WasRead:
    def __init__(self):
        self.saved = []   # [(id, shape, read)]

    def __enter__(self):
        def pack(t):
            rec = [t, False]
            self.saved.append(rec)
            return rec

        def unpack(rec):
            rec[1] = True
            return rec[0]

        self._ctx = torch.autograd.graph.saved_tensors_hooks(pack, unpack)
        self._ctx.__enter__()
        return self

    def __exit__(self, *a):
        self._ctx.__exit__(*a)


def _m(shape, rg, dtype=BF):
    return torch.empty(shape, device="meta", dtype=dtype).requires_grad_(bool(rg))


def _run(fwd, leaves):
    with _WasRead() as wr:
        out = fwd()
        if isinstance(out, tuple):
            out = out[0]
        if out.requires_grad:
            out.sum().backward()
    return wr.saved


FLAGS = list(itertools.product([0, 1], repeat=3))


def _check(saved, x, w, x_rg, w_rg):
    unread = [tuple(t.shape) for t, read in saved if not read]
    assert not unread, f"saved but never read by backward: {unread}"
    fulls = [t for t, _ in saved]
    if any(t is x for t in fulls):
        assert w_rg, "x kept although dW was not requested"
    if w is not None and any(t is w for t in fulls):
        assert x_rg, "W kept although dX was not requested"


@pytest.mark.parametrize("flags", FLAGS)
def test_linear_minimal(flags):
    x_rg, w_rg, b_rg = flags
    x, w, b = _m((4, 6, 8), x_rg), _m((5, 8), w_rg), _m((5,), b_rg)
    saved = _run(lambda: MF.linear(x, w, b), (x, w, b))
    _check(saved, x, w, x_rg, w_rg)


@pytest.mark.parametrize("flags", FLAGS)
def test_conv2d_minimal(flags):
    x_rg, w_rg, b_rg = flags
    x, w, b = _m((2, 8, 9, 9), x_rg), _m((16, 8, 3, 3), w_rg), _m((16,), b_rg)
    saved = _run(lambda: MF.conv2d(x, w, b, 2, 1), (x, w, b))
    _check(saved, x, w, x_rg, w_rg)


@pytest.mark.parametrize("flags", FLAGS)
def test_conv_transpose2d_minimal(flags):
    x_rg, w_rg, b_rg = flags
    x, w, b = _m((2, 8, 5, 5), x_rg), _m((8, 16, 3, 3), w_rg), _m((16,), b_rg)
    saved = _run(lambda: MF.conv_transpose2d(x, w, b, 2, 1, 1), (x, w, b))
    _check(saved, x, w, x_rg, w_rg)


@pytest.mark.parametrize("flags", FLAGS)
def test_batchnorm_eval_minimal(flags):
    x_rg, w_rg, b_rg = flags
    x, w, b = _m((2, 8, 5, 5), x_rg), _m((8,), w_rg, torch.float32), _m((8,), b_rg, torch.float32)
    rm, rv = torch.empty(8, device="meta"), torch.empty(8, device="meta")
    saved = _run(lambda: MF.batch_norm_eval(x, rm, rv, w, b, 1e-5), (x, w, b))
    _check(saved, x, w, x_rg, w_rg)
    # running statistics are module state, never tape state
    assert not any(t is rm or t is rv for t, _ in saved)


@pytest.mark.parametrize("flags", FLAGS)
def test_batchnorm_relu_minimal(flags):
    x_rg, w_rg, b_rg = flags
    x, w, b = _m((2, 8, 5, 5), x_rg), _m((8,), w_rg, torch.float32), _m((8,), b_rg, torch.float32)
    bn = nn.BatchNorm2d(8).to("meta").eval()
    bn.weight, bn.bias = nn.Parameter(w, bool(w_rg)), nn.Parameter(b, bool(b_rg))
    xs = x.contiguous(memory_format=torch.channels_last)
    saved = _run(lambda: MF.batch_norm_relu_eval(xs, bn), (x,))
    _check(saved, xs, bn.weight, x_rg, w_rg)


@pytest.mark.parametrize("flags", FLAGS)
def test_layernorm_minimal(flags):
    x_rg, w_rg, b_rg = flags
    x, w, b = _m((3, 7, 16), x_rg), _m((16,), w_rg), _m((16,), b_rg)
    saved = _run(lambda: MF.layer_norm(x, (16,), w, b), (x, w, b))
    unread = [tuple(t.shape) for t, read in saved if not read]
    assert not unread
    # LayerNorm row (rules.py:89-96): x and stats iff x or w needs a grad, w iff x does
    fulls = [t for t, _ in saved]
    assert any(t is x for t in fulls) == bool(x_rg or w_rg)
    assert any(t is w for t in fulls) == bool(x_rg)


@pytest.mark.parametrize("rg", [0, 1])
def test_relu_pool_dropout_minimal(rg):
    x = _m((2, 8, 6, 6), rg)
    for fwd in (lambda: MF.relu(x), lambda: MF.max_pool2d(x, 3, 2, 1),
                lambda: MF.dropout(x, 0.1, True, seed=1)):
        saved = _run(fwd, (x,))
        assert all(read for _, read in saved)
        if not rg:
            assert saved == []  # output needs no grad: nothing kept at all
        # never the activation itself: a bit mask / index map / RNG key only
        assert not any(t is x for t, _ in saved)


@pytest.mark.parametrize("flags", FLAGS)
def test_fused_conv_bn_relu_minimal(flags):
    x_rg, w_rg, _ = flags
    conv = pnn.MemSaveConv2d(16, 16, 3, padding=1, bias=False).to("meta", BF)
    conv.weight.requires_grad_(bool(w_rg))
    bn = nn.BatchNorm2d(16).to("meta", BF).eval().requires_grad_(False)
    x = _m((2, 16, 6, 6), x_rg).contiguous(memory_format=torch.channels_last)
    saved = _run(lambda: MF.conv_bn_relu(x, conv, bn, True), (x,))
    _check(saved, x, conv.weight, x_rg, w_rg)
