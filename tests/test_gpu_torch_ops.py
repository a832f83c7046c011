"""The PyTorch custom-op boundary (torch.ops.memsave, csrc/torch_ops.cpp) on
the GPU: torch.compile traces the converted model without a graph break inside
the layers, a CUDA graph of a whole fwd+bwd step replays and matches eager, and
the saved set under both is unchanged."""

import pytest
import torch
from torch import nn

from paper_2404_12406_b200 import launch_count
from paper_2404_12406_b200.nn import convert_to_memory_saving

pytestmark = pytest.mark.gpu

DEV = "cuda"
CL = torch.channels_last


def _resnet18(fuse):
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.resnet18()
    g = torch.Generator().manual_seed(0)
    for mod in m.modules():
        if isinstance(mod, nn.BatchNorm2d):
            mod.running_mean.copy_(torch.randn(mod.num_features, generator=g) * 0.1)
            mod.running_var.copy_(torch.rand(mod.num_features, generator=g) * 1.5 + 0.5)
    m = m.to(DEV, torch.bfloat16).to(memory_format=CL).eval().requires_grad_(False)
    return convert_to_memory_saving(m, fuse=fuse)


def _batch(n=4, hw=64, seed=1):
    gen = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn((n, 3, hw, hw), generator=gen, device=DEV).to(torch.bfloat16)
    y = torch.randint(0, 1000, (n,), generator=gen, device=DEV)
    return x.contiguous(memory_format=CL), y


def _eager_step(model, x, y):
    x = x.detach().clone().requires_grad_(True)
    loss = nn.functional.cross_entropy(model(x).float(), y)
    loss.backward()
    return loss.detach(), x.grad


def test_torch_compile_fullgraph_no_break():
    from torch._dynamo.utils import counters
    torch._dynamo.reset()
    counters.clear()
    model = _resnet18(fuse=False)
    x, y = _batch()
    ref_loss, ref_grad = _eager_step(model, x, y)

    def step(inp, tgt):
        return nn.functional.cross_entropy(model(inp).float(), tgt)

    cstep = torch.compile(step, backend="aot_eager", fullgraph=True)
    xc = x.detach().clone().requires_grad_(True)
    n0 = launch_count()
    loss = cstep(xc, y)
    loss.backward()
    torch.cuda.synchronize()
    assert launch_count() > n0  # the compiled graph runs our kernels (opaque custom ops)
    assert not counters["graph_break"], dict(counters["graph_break"])
    torch.testing.assert_close(loss, ref_loss, rtol=0, atol=0)
    torch.testing.assert_close(xc.grad, ref_grad, rtol=0, atol=0)


def test_torch_compile_fused_graph_runs():
    torch._dynamo.reset()
    model = _resnet18(fuse=True)
    x, y = _batch(seed=3)
    ref_loss, ref_grad = _eager_step(model, x, y)
    cmodel = torch.compile(model, backend="aot_eager")
    xc = x.detach().clone().requires_grad_(True)
    loss = nn.functional.cross_entropy(cmodel(xc).float(), y)
    loss.backward()
    torch.testing.assert_close(loss.detach(), ref_loss, rtol=0, atol=0)
    torch.testing.assert_close(xc.grad, ref_grad, rtol=0, atol=0)


@pytest.mark.parametrize("fuse", [False, True])
def test_cuda_graph_capture_of_a_step(fuse):
    model = _resnet18(fuse=fuse)
    x0, y = _batch(seed=5)
    x1, _ = _batch(seed=6)
    static_x = x0.detach().clone().requires_grad_(True)

    def step():
        static_x.grad = None
        loss = nn.functional.cross_entropy(model(static_x).float(), y)
        loss.backward()
        return loss

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            step()
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    static_x.grad = None
    with torch.cuda.graph(graph):
        static_loss = nn.functional.cross_entropy(model(static_x).float(), y)
        static_loss.backward()
    for xin in (x1, x0):
        with torch.no_grad():
            static_x.copy_(xin)
        n0 = launch_count()
        graph.replay()
        torch.cuda.synchronize()
        assert launch_count() == n0  # replays launch nothing from the host
        ref_loss, ref_grad = _eager_step(model, xin, y)
        torch.testing.assert_close(static_loss.detach(), ref_loss, rtol=0, atol=0)
        torch.testing.assert_close(static_x.grad, ref_grad, rtol=0, atol=0)


def test_saved_set_through_the_op_layer():
    """x kept only for dW, W only for dX, on CUDA through torch.ops.memsave."""
    from paper_2404_12406_b200 import functional as MF
    for x_rg, w_rg in ((True, False), (False, True), (True, True)):
        x = torch.randn(8, 64, device=DEV, dtype=torch.bfloat16).requires_grad_(x_rg)
        w = torch.randn(32, 64, device=DEV, dtype=torch.bfloat16).requires_grad_(w_rg)
        saved = []
        with torch.autograd.graph.saved_tensors_hooks(lambda t: saved.append(t) or t,
                                                      lambda t: t):
            MF.linear(x, w)
        assert any(t is x for t in saved) == w_rg
        assert any(t is w for t in saved) == x_rg


@pytest.mark.gpu
def test_bert_fused_output_projection_matches_unfused():
    """A small BERT in train mode (dropout 0.1) converted with fuse=True (the
    attention-output and output blocks become Linear -> dropout -> + residual
    nodes) gives the same logits, bit for bit, as the unfused memsave model
    under the same seeds, and the same trainable-bias gradients (up to the
    order of the fp32 atomics in the column sums)."""
    import copy

    from transformers import BertConfig, BertForSequenceClassification

    from paper_2404_12406_b200.nn import convert_to_memory_saving
    torch.manual_seed(0)
    cfg = BertConfig(num_hidden_layers=2, hidden_size=128, num_attention_heads=2,
                     intermediate_size=256, attn_implementation="sdpa")
    base = BertForSequenceClassification(cfg).to("cuda", torch.bfloat16).train()
    for name, p in base.named_parameters():
        p.requires_grad_(name.startswith("classifier.") or (
            ".attention." in name and name.endswith(".bias") and "LayerNorm" not in name))
    a = convert_to_memory_saving(copy.deepcopy(base), fuse=False)
    b = convert_to_memory_saving(copy.deepcopy(base), fuse=True)
    assert isinstance(b.bert.encoder.layer[0].output, torch.fx.GraphModule)
    ids = torch.randint(0, cfg.vocab_size, (4, 64), device="cuda")
    outs = []
    for m in (a, b):
        torch.manual_seed(123)
        logits = m(input_ids=ids).logits
        logits.float().square().sum().backward()
        outs.append((logits.detach(), {n: p.grad for n, p in m.named_parameters()
                                       if p.requires_grad}))
    assert torch.equal(outs[0][0], outs[1][0])
    assert outs[0][1].keys() == outs[1][1].keys()
    for n in outs[0][1]:
        torch.testing.assert_close(outs[0][1][n], outs[1][1][n], rtol=2 ** -6, atol=1e-3,
                                   msg=n)
