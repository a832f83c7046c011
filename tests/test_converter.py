"""convert_to_memory_saving: kind filter, idempotence, parameter sharing,
state_dict compatibility, unsupported variants untouched."""

import torch
from torch import nn

import memsave_torch.nn as mnn
from paper_2404_12406_b200.nn import (MemSaveBatchNorm2d, MemSaveConv2d, MemSaveLinear,
                                      convert_to_memory_saving)


def _net():
    return nn.Sequential(
        nn.Conv2d(3, 8, 3, padding=1, bias=False), nn.BatchNorm2d(8), nn.ReLU(),
        nn.Sequential(nn.Conv2d(8, 8, 3, padding=1), nn.BatchNorm2d(8)),
        nn.Conv2d(8, 8, 3, padding=2, dilation=2),       # dilation: unsupported
        nn.Conv2d(8, 8, 3, padding=1, groups=2),         # groups: unsupported
        nn.Flatten(), nn.Linear(8 * 4 * 4, 10))


def test_alias_package_exports_same_objects():
    assert mnn.convert_to_memory_saving is convert_to_memory_saving
    assert mnn.MemSaveConv2d is MemSaveConv2d


def test_convert_all_and_unsupported_untouched():
    net = _net()
    sd = {k: v.clone() for k, v in net.state_dict().items()}
    params = [p for p in net.parameters()]
    out = convert_to_memory_saving(net)
    assert out is net
    kinds = [type(m).__name__ for m in net.modules()]
    assert kinds.count("MemSaveConv2d") == 2
    assert kinds.count("MemSaveBatchNorm2d") == 2
    assert kinds.count("MemSaveLinear") == 1
    assert kinds.count("Conv2d") == 2  # dilated + grouped left alone
    # parameters are shared, not copied: optimiser references stay valid
    assert [id(p) for p in net.parameters()] == [id(p) for p in params]
    # identical state_dict keys and values
    sd2 = net.state_dict()
    assert list(sd2) == list(sd)
    for k in sd:
        assert torch.equal(sd[k], sd2[k])


def test_convert_is_idempotent():
    net = convert_to_memory_saving(_net())
    before = [(n, type(m)) for n, m in net.named_modules()]
    convert_to_memory_saving(net)
    assert [(n, type(m)) for n, m in net.named_modules()] == before


def test_kind_filter():
    net = convert_to_memory_saving(_net(), linear=False, batchnorm2d=False)
    kinds = [type(m).__name__ for m in net.modules()]
    assert "MemSaveConv2d" in kinds and "MemSaveLinear" not in kinds
    assert "MemSaveBatchNorm2d" not in kinds


def test_top_level_module_is_returned_converted():
    lin = nn.Linear(4, 3)
    out = convert_to_memory_saving(lin)
    assert isinstance(out, MemSaveLinear) and out.weight is lin.weight


def test_clone_params():
    conv = nn.Conv2d(4, 4, 3)
    m = MemSaveConv2d.from_nn_Conv2d(conv, clone_params=True)
    assert m.weight is not conv.weight and torch.equal(m.weight, conv.weight)


def test_bn_buffers_shared_and_train_mode_is_stock():
    bn = nn.BatchNorm2d(4)
    m = MemSaveBatchNorm2d.from_nn_BatchNorm2d(bn)
    assert m.running_mean is bn.running_mean and m.running_var is bn.running_var
    m.train()
    x = torch.randn(3, 4, 5, 5)
    ref = nn.BatchNorm2d(4)
    torch.testing.assert_close(m(x), ref(x))  # training mode: stock semantics, stats updated
    torch.testing.assert_close(m.running_mean, ref.running_mean)


def test_cpu_tensors_fail_loudly():
    import pytest
    m = MemSaveLinear(4, 3)
    with pytest.raises(RuntimeError, match="no CPU path"):
        m(torch.randn(2, 4))


class _Act(nn.Module):  # an activation wrapper that fx traces through (HF style)
    def forward(self, x):
        return nn.functional.gelu(x)


class _Intermediate(nn.Module):
    def __init__(self):
        super().__init__()
        self.dense = nn.Linear(8, 16)
        self.act = _Act()

    def forward(self, h):
        return self.act(self.dense(h))


class _Block(nn.Module):
    def __init__(self):
        super().__init__()
        self.inter = _Intermediate()
        self.out = nn.Linear(16, 8)
        self.tanh_mlp = nn.Sequential(nn.Linear(8, 8), nn.GELU(approximate="tanh"))

    def forward(self, x, mask=None):  # optional argument: not traced as a whole
        if mask is not None:
            x = x * mask
        return self.out(self.inter(x)) + self.tanh_mlp(x)


def test_fuse_linear_gelu_per_module():
    from paper_2404_12406_b200.nn import fuse_linear_gelu
    torch.manual_seed(0)
    net = _Block()
    sd = {k: v.clone() for k, v in net.state_dict().items()}
    convert_to_memory_saving(net, fuse=True)
    assert not isinstance(net.inter, torch.fx.GraphModule)  # opt-in pass
    fuse_linear_gelu(net)
    code = net.inter.code
    assert "_gelu_layer" in code and "gelu(" not in code.replace("_gelu_layer", "")
    # the tanh GELU and the module with an optional argument are left alone
    assert type(net.tanh_mlp) is nn.Sequential and isinstance(net.tanh_mlp[1], nn.GELU)
    assert not isinstance(net, torch.fx.GraphModule)
    assert net.state_dict().keys() == sd.keys()
    assert all(torch.equal(net.state_dict()[k], v) for k, v in sd.items())
    # idempotent: a second pass finds nothing more
    assert fuse_linear_gelu(net) is net
    # shapes and gradients flow on meta
    mnet = _Block().to("meta")
    fuse_linear_gelu(convert_to_memory_saving(mnet))
    x = torch.empty(4, 8, device="meta", requires_grad=True)
    mnet(x).sum().backward()
    assert x.grad.shape == x.shape and mnet.inter.dense.weight.grad.shape == (16, 8)


def test_fuse_linear_gelu_bert_intermediate_blocks():
    from transformers import BertConfig, BertForSequenceClassification

    from paper_2404_12406_b200.nn import fuse_linear_gelu
    cfg = BertConfig(num_hidden_layers=2, hidden_size=64, num_attention_heads=2,
                     intermediate_size=128, attn_implementation="sdpa")
    with torch.device("meta"):
        m = BertForSequenceClassification(cfg)
    keys = list(m.state_dict().keys())
    m = fuse_linear_gelu(convert_to_memory_saving(m, fuse=True))
    for layer in m.bert.encoder.layer:
        assert isinstance(layer.intermediate, torch.fx.GraphModule)
        assert "_gelu_layer" in layer.intermediate.code
        assert type(layer.output.dense) is MemSaveLinear
    assert list(m.state_dict().keys()) == keys
    ids = torch.zeros(2, 16, dtype=torch.long, device="meta")
    m(input_ids=ids).logits.sum().backward()


def test_fuse_linear_dropout_add_bert_output_blocks():
    """convert_to_memory_saving(fuse=True) turns BERT's attention-output and
    output blocks (dense -> dropout -> + input -> LayerNorm) into the fused node;
    parameters, state_dict keys and the train/eval switch are kept."""
    from transformers import BertConfig, BertForSequenceClassification
    cfg = BertConfig(num_hidden_layers=2, hidden_size=64, num_attention_heads=2,
                     intermediate_size=128, attn_implementation="sdpa")
    with torch.device("meta"):
        m = BertForSequenceClassification(cfg)
    keys = list(m.state_dict().keys())
    m = convert_to_memory_saving(m, fuse=True)
    for layer in m.bert.encoder.layer:
        for blk in (layer.attention.output, layer.output):
            assert isinstance(blk, torch.fx.GraphModule)
            assert "_dropout_add_layer" in blk.code
        assert not isinstance(layer.intermediate, torch.fx.GraphModule)
    assert list(m.state_dict().keys()) == keys
    m.eval()
    assert not m.bert.encoder.layer[0].output.dropout.training
    ids = torch.zeros(2, 16, dtype=torch.long, device="meta")
    m.train()
    m(input_ids=ids).logits.sum().backward()
    # converting without dropout leaves the blocks alone
    with torch.device("meta"):
        m2 = BertForSequenceClassification(cfg)
    convert_to_memory_saving(m2, fuse=True, dropout=False)
    assert not isinstance(m2.bert.encoder.layer[0].output, torch.fx.GraphModule)
