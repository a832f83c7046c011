"""Semantics of the fx fusion pass and the fused-conv entry point on the meta
device (no GPU): kind filters, residual shape guard, tee only for a
differentiable input, in-place consumers of fused outputs, and the
``memsave_torch.nn`` alias surface."""

import operator

import pytest
import torch
from torch import nn

import memsave_torch.nn as mnn
import paper_2404_12406_b200.nn as pnn
from paper_2404_12406_b200 import functional as MF
from paper_2404_12406_b200.nn import convert_to_memory_saving


def _meta_resnet_block():
    class Block(nn.Module):
        def __init__(self):
            super().__init__()
            self.conv1 = nn.Conv2d(64, 64, 3, padding=1, bias=False)
            self.bn1 = nn.BatchNorm2d(64)
            self.relu = nn.ReLU()
            self.conv2 = nn.Conv2d(64, 64, 3, padding=1, bias=False)
            self.bn2 = nn.BatchNorm2d(64)

        def forward(self, x):
            y = self.relu(self.bn1(self.conv1(x)))
            y = self.bn2(self.conv2(y))
            return self.relu(y + x)

    return Block().to(device="meta", dtype=torch.bfloat16).eval().requires_grad_(False)


def _fused_calls(gm):
    return [n for n in gm.graph.nodes if n.op == "call_function" and n.target is MF.fused_conv]


def test_alias_exports_every_layer():
    for name in pnn.__all__:
        assert getattr(mnn, name) is getattr(pnn, name)


@pytest.mark.parametrize("kind", ["conv2d", "batchnorm2d", "relu"])
def test_fx_pass_honours_kind_filter(kind):
    full = convert_to_memory_saving(_meta_resnet_block(), fuse=True)
    assert len(_fused_calls(full)) == 2
    gm = convert_to_memory_saving(_meta_resnet_block(), fuse=True, **{kind: False})
    calls = _fused_calls(gm) if isinstance(gm, torch.fx.GraphModule) else []
    if kind == "conv2d":
        assert calls == []  # stock convs are never fused into the memsave kernel
    elif kind == "batchnorm2d":
        assert all(c.args[2] is None for c in calls)
        mods = dict(gm.named_modules())
        assert sum(type(m) is nn.BatchNorm2d for m in mods.values()) == 2
    else:
        # no ReLU folded into a fused conv and no add->relu rewrite
        assert all(c.args[3] is False for c in calls)
        assert not any(n.target is MF.add_relu for n in gm.graph.nodes)


def test_residual_shape_mismatch_falls_back_to_broadcasting_add():
    conv = pnn.MemSaveConv2d(64, 64, 3, padding=1, bias=False).to("meta", torch.bfloat16)
    bn = nn.BatchNorm2d(64).to("meta", torch.bfloat16).eval().requires_grad_(False)
    conv.requires_grad_(False)
    x = torch.empty(4, 64, 8, 8, device="meta", dtype=torch.bfloat16)
    calls = []
    orig = MF._ConvBNFn.apply

    def spy(*a):
        calls.append(a[3])
        return orig(*a)

    MF._ConvBNFn.apply = spy
    try:
        r_bcast = torch.empty(1, 64, 8, 8, device="meta", dtype=torch.bfloat16)
        y, _, _ = MF.fused_conv(x, conv, bn, True, residual=r_bcast)
        assert tuple(y.shape) == (4, 64, 8, 8)
        assert all(r is None for r in calls)  # the epilogue never saw the residual
        calls.clear()
        r_full = torch.empty(4, 64, 8, 8, device="meta", dtype=torch.bfloat16)
        MF.fused_conv(x, conv, bn, True, residual=r_full)
        assert len(calls) == 1 and calls[0] is r_full
    finally:
        MF._ConvBNFn.apply = orig


def test_tee_of_non_differentiable_input_is_the_input_itself():
    conv = pnn.MemSaveConv2d(64, 64, 3, padding=1, bias=False).to("meta", torch.bfloat16)
    bn = nn.BatchNorm2d(64).to("meta", torch.bfloat16).eval().requires_grad_(False)
    conv.weight.requires_grad_(True)  # fine-tuning this conv only
    x = torch.empty(2, 64, 8, 8, device="meta", dtype=torch.bfloat16)
    y, _, alias = MF.fused_conv(x, conv, bn, True, tee=True)
    assert alias is x and not alias.requires_grad
    # x that needs a grad: the alias carries the second gradient into dgrad
    xg = x.clone().requires_grad_(True)
    _, _, alias2 = MF.fused_conv(xg, conv, bn, True, tee=True)
    assert alias2 is not xg and alias2.requires_grad


def test_inplace_consumer_of_fused_output_is_legal():
    conv = pnn.MemSaveConv2d(64, 64, 3, padding=1, bias=False).to("meta", torch.bfloat16)
    bn = nn.BatchNorm2d(64).to("meta", torch.bfloat16).eval().requires_grad_(False)
    conv.requires_grad_(False)
    x = torch.empty(2, 64, 8, 8, device="meta", dtype=torch.bfloat16, requires_grad=True)
    y = MF.conv_bn_relu(x, conv, bn, True)
    y.add_(1.0)  # was: "a view ... is being modified inplace"
    y.relu_()
    y.sum().backward()
    assert x.grad is not None and x.grad.shape == x.shape


def test_fused_block_graph_has_tee_and_deferred_relu():
    gm = convert_to_memory_saving(_meta_resnet_block(), fuse=True)
    calls = _fused_calls(gm)
    assert any(c.kwargs.get("tee") for c in calls)
    assert any("in_mask" in c.kwargs for c in calls)
    assert any(n.target is operator.getitem and n.args[1] == 2 for n in gm.graph.nodes)
