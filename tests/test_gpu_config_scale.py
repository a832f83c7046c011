"""Config-scale parity: the sm_100a kernels at the BASELINE.json configs' real
shapes against the float64 oracle (oracle/, SURVEY.md §8(c) tolerances).

Full-size f64 oracles of these shapes would take minutes on the host, so every
check evaluates the oracle exactly on a seeded SUBSET of the outputs: whole
output rows for forward and dX (each row is a complete K-long reduction), and
an (n, k) block of dW computed from the full M-long reduction (every row of X
and dY enters it).  The inputs are drawn on the GPU in bf16 and only the slices
the oracle needs are copied back.

Shapes:
  BERT-base b64 s512: M = 32768; 768->768, 768->3072, 3072->768
  Llama-3-8B b2 s2048: M = 4096; 4096->4096, 4096->1024, 4096->14336,
                       14336->4096 (last-wave K split), lm_head 4096->128256
  VGG-16 block 4 / ResNet-101 layer 4 conv wgrad (long pixel reductions)
  Fig. 1 layer-1 dW at the full (32, 8, 256, 256) fp32 input (2.1 M-term reduction)

Then a layer-by-layer ResNet-18 / VGG-16 forward + backward: every MemSave
module's output, input gradient and weight gradient against the oracle applied
to that module's own GPU input / output gradient (reference numpy_impl.py:12-78,
SPEC.md:241-274)."""

import numpy as np
import pytest
import torch

import oracle
from paper_2404_12406_b200 import functional as MF
from paper_2404_12406_b200 import launch_stats

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _np(t):
    return np.ascontiguousarray(t.detach().float().cpu().double().numpy())


def _bf16_close(a, ref64, what, ulps=1.01):
    oracle.assert_close_lowp(_np(a) if isinstance(a, torch.Tensor) else a, ref64, "bf16",
                             ulps=ulps, what=what)


def _randn(shape, gen, scale=1.0, dtype=torch.bfloat16):
    return (torch.randn(shape, generator=gen, device=DEV, dtype=torch.float32) * scale).to(dtype)


LINEAR_SHAPES = [
    # (tag, M, K, N)
    ("bert_qkvo", 32768, 768, 768),
    ("bert_ffn_up", 32768, 768, 3072),
    ("bert_ffn_down", 32768, 3072, 768),
    ("llama_q_o", 4096, 4096, 4096),
    ("llama_kv", 4096, 4096, 1024),
    ("llama_gate_up", 4096, 4096, 14336),
    ("llama_down", 4096, 14336, 4096),
    ("llama_lm_head", 4096, 4096, 128256),
]


@pytest.mark.parametrize("tag,M,K,N", LINEAR_SHAPES, ids=[s[0] for s in LINEAR_SHAPES])
def test_linear_config_shapes(tag, M, K, N):
    gen = torch.Generator(device=DEV).manual_seed(M + 7 * K + N)
    x = _randn((M, K), gen).requires_grad_(True)
    w = _randn((N, K), gen, scale=K ** -0.5).requires_grad_(True)
    b = _randn((N,), gen).requires_grad_(True)
    g = _randn((M, N), gen)
    u0 = launch_stats()["umma"]
    y = MF.linear(x, w, b)
    y.backward(g)
    torch.cuda.synchronize()
    assert launch_stats()["umma"] - u0 >= 3  # fwd, dX, dW on the tcgen05 kernels
    rs = np.random.default_rng(M ^ N)
    rows = np.sort(rs.choice(M, size=96, replace=False))
    ncols = np.sort(rs.choice(N, size=min(N, 64), replace=False))
    kcols = np.sort(rs.choice(K, size=min(K, 64), replace=False))
    ri = torch.as_tensor(rows, device=DEV)
    wq = _np(w)
    xr = _np(x[ri])
    gr = _np(g[ri])
    # forward rows: full K-long reductions
    _bf16_close(y[ri], oracle.linear_fwd(xr, wq, _np(b)), f"{tag} y")
    # dX rows: full N-long reductions
    _bf16_close(x.grad[ri], oracle.linear_dx(gr, wq), f"{tag} dx")
    # dW block: full M-long reductions over every row of X and dY
    ni, ki = torch.as_tensor(ncols, device=DEV), torch.as_tensor(kcols, device=DEV)
    dw_ref = oracle.linear_dw(_np(x[:, ki]), _np(g[:, ni]))
    _bf16_close(w.grad[ni][:, ki], dw_ref, f"{tag} dW")
    _bf16_close(b.grad[ni], oracle.linear_db(_np(g[:, ni])), f"{tag} db")


CONV_WGRAD = [
    # (tag, n, c, h, k, r, stride, pad)
    ("vgg16_conv4_1", 32, 256, 28, 512, 3, 1, 1),
    ("vgg16_conv4_2", 32, 512, 28, 512, 3, 1, 1),
    ("vgg16_conv5_x", 64, 512, 14, 512, 3, 1, 1),
    ("r101_l4_conv1", 128, 2048, 7, 512, 1, 1, 0),
    ("r101_l4_conv2", 128, 512, 7, 512, 3, 1, 1),
    ("r101_l4_conv3", 128, 512, 7, 2048, 1, 1, 0),
]


@pytest.mark.parametrize("tag,n,c,h,k,r,s,p", CONV_WGRAD, ids=[t[0] for t in CONV_WGRAD])
def test_conv_wgrad_long_reduction(tag, n, c, h, k, r, s, p):
    gen = torch.Generator(device=DEV).manual_seed(n * c + k)
    cl = torch.channels_last
    x = _randn((n, c, h, h), gen).contiguous(memory_format=cl)
    w = _randn((k, c, r, r), gen, scale=(c * r * r) ** -0.5).contiguous(memory_format=cl)
    w.requires_grad_(True)
    oh = (h + 2 * p - r) // s + 1
    g = _randn((n, k, oh, oh), gen).contiguous(memory_format=cl)
    y = MF.conv2d(x, w, None, s, p)
    y.backward(g)
    torch.cuda.synchronize()
    rs = np.random.default_rng(c + k)
    ks = np.sort(rs.choice(k, size=8, replace=False))
    ki = torch.as_tensor(ks, device=DEV)
    ref = oracle.conv2d_dw(_np(x), _np(g[:, ki]), s, p, r, r)  # every pixel of the batch
    _bf16_close(w.grad[ki], ref, f"{tag} dW")
    # forward rows at this scale too (one image's output pixels for the sampled k)
    _bf16_close(y[:1, ki], oracle.conv2d_fwd(_np(x[:1]), _np(w[ki]), s, p), f"{tag} y")


def test_fig1_full_size_dw_fp32():
    """Fig. 1 layer 1: dW over the full (32, 8, 256, 256) fp32 input, 2.1 M terms per
    output (numba_impl.py:57-75 accumulates it sequentially in f32; the oracle is f64)."""
    gen = torch.Generator(device=DEV).manual_seed(32)
    x = torch.randn((32, 8, 256, 256), generator=gen, device=DEV)
    w = (torch.randn((8, 8, 3, 3), generator=gen, device=DEV) / 24).requires_grad_(True)
    g = torch.randn((32, 8, 256, 256), generator=gen, device=DEV)
    y = MF.conv2d(x, w, None, 1, 1)
    y.backward(g)
    torch.cuda.synchronize()
    xq, gq = _np(x), _np(g)
    oracle.assert_close_fp32(_np(w.grad), oracle.conv2d_dw(xq, gq, 1, 1, 3, 3), what="fig1 dW")
    oracle.assert_close_fp32(_np(y[:2]), oracle.conv2d_fwd(xq[:2], _np(w), 1, 1), what="fig1 y")


# ------------------------------------------------------------------ layer by layer
def _module_oracle(mod, x, gy):
    """(y, dx, dW or None) of one MemSave module by the oracle, f64 on the GPU's
    own (bf16) input and output gradient."""
    import paper_2404_12406_b200.nn as pnn
    if isinstance(mod, pnn.MemSaveConv2d):
        w = _np(mod.weight)
        s, p = mod.stride[0], mod.padding[0]
        y = oracle.conv2d_fwd(x, w, s, p)
        if mod.bias is not None:
            y = y + _np(mod.bias)[None, :, None, None]
        dx = oracle.conv2d_dx(gy, w, s, p, x.shape[2], x.shape[3])
        dw = oracle.conv2d_dw(x, gy, s, p, w.shape[2], w.shape[3]) \
            if mod.weight.requires_grad else None
        return y, dx, dw
    if isinstance(mod, pnn.MemSaveBatchNorm2d):
        m, v = _np(mod.running_mean), _np(mod.running_var)
        wt, bt = _np(mod.weight), _np(mod.bias)
        return (oracle.bn_eval_fwd(x, m, v, wt, bt, mod.eps), oracle.bn_eval_dx(gy, v, wt, mod.eps),
                oracle.bn_eval_dw(gy, x, m, v, mod.eps) if mod.weight.requires_grad else None)
    if isinstance(mod, pnn.MemSaveReLU):
        y, mask = oracle.relu_fwd(x)
        return y, oracle.relu_bwd(gy, mask), None
    if isinstance(mod, pnn.MemSaveMaxPool2d):
        k, s, p = mod.kernel_size, mod.stride, mod.padding
        k, s, p = [(v, v) if isinstance(v, int) else v for v in (k, s, p)]
        y, _local, flat = oracle.maxpool2d_fwd(x, k[0], k[1], s[0], s[1], p[0], p[1])
        return y, oracle.maxpool2d_bwd(gy, flat, x.shape[2], x.shape[3]), None
    if isinstance(mod, pnn.MemSaveLinear):
        w = _np(mod.weight)
        y = oracle.linear_fwd(x, w, None if mod.bias is None else _np(mod.bias))
        return y, oracle.linear_dx(gy, w), (oracle.linear_dw(x, gy)
                                            if mod.weight.requires_grad else None)
    return None


class _Tap(torch.autograd.Function):
    """Identity that copies its input (so in-place consumers stay legal) and
    records the gradient that flows back through it."""

    @staticmethod
    def forward(ctx, x, store, key):
        ctx.store, ctx.key = store, key
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        ctx.store[ctx.key] = g.detach().clone()
        return g, None, None


def _layer_by_layer(model, x, tag):
    """Run the converted model once; every MemSave module's input is tapped in
    front of it (its own input gradient) and its output behind it (the gradient
    arriving from the rest of the network)."""
    import paper_2404_12406_b200.nn as pnn
    from paper_2404_12406_b200.nn import convert_to_memory_saving
    model = convert_to_memory_saving(model)
    calls, grads = [], {}   # one entry per module CALL (a ResNet block reuses its ReLU)
    open_call = {}
    hooks = []
    for name, m in model.named_modules():
        if not isinstance(m, pnn._MEMSAVE_TYPES):
            continue

        def pre_hook(mod, inp, name=name):
            i = len(calls)
            calls.append({"name": name, "x": inp[0].detach().clone()})
            open_call[name] = i
            if inp[0].requires_grad:
                return (_Tap.apply(inp[0], grads, (i, "gx")),) + tuple(inp[1:])
            return None

        def fwd_hook(mod, inp, out, name=name):
            i = open_call[name]
            calls[i]["y"] = out.detach().clone()
            if out.requires_grad:
                return _Tap.apply(out, grads, (i, "gy"))
            return None

        hooks += [m.register_forward_pre_hook(pre_hook), m.register_forward_hook(fwd_hook)]
    out = model(x)
    gen = torch.Generator(device=DEV).manual_seed(5)
    out.backward(torch.randn(out.shape, generator=gen, device=DEV).to(out.dtype))
    torch.cuda.synchronize()
    for h in hooks:
        h.remove()
    checked = 0
    mods = dict(model.named_modules())
    ncalls = {}
    for c in calls:
        ncalls[c["name"]] = ncalls.get(c["name"], 0) + 1
    for i, r in enumerate(calls):
        name = r["name"]
        mod = mods[name]
        gy_t = grads.get((i, "gy"))
        gy = _np(gy_t) if gy_t is not None else np.zeros(r["y"].shape)
        res = _module_oracle(mod, _np(r["x"]), gy)
        if res is None:
            continue
        y_ref, dx_ref, dw_ref = res
        ulps = 2.01 if isinstance(mod, pnn.MemSaveBatchNorm2d) else 1.01
        _bf16_close(r["y"], y_ref, f"{tag}.{name}#{i} y", ulps)
        gx = grads.get((i, "gx"))
        if gx is not None:
            _bf16_close(gx, dx_ref, f"{tag}.{name}#{i} dx", ulps)
        if dw_ref is not None and ncalls[name] == 1:
            _bf16_close(mod.weight.grad, dw_ref, f"{tag}.{name} dW", ulps)
        checked += 1
    return checked


def test_resnet18_layer_by_layer_vs_oracle():
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.resnet18()
    g = torch.Generator().manual_seed(0)
    for mod in m.modules():
        if isinstance(mod, torch.nn.BatchNorm2d):
            mod.running_mean.copy_(torch.randn(mod.num_features, generator=g) * 0.1)
            mod.running_var.copy_(torch.rand(mod.num_features, generator=g) * 1.5 + 0.5)
    m = m.to(DEV, torch.bfloat16).to(memory_format=torch.channels_last).eval()
    m.requires_grad_(False)
    m.layer4.requires_grad_(True)  # dW checks on the last stage too
    gen = torch.Generator(device=DEV).manual_seed(1)
    x = torch.randn((2, 3, 112, 112), generator=gen, device=DEV).to(torch.bfloat16)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    n = _layer_by_layer(m, x, "resnet18")
    assert n >= 50, n


def test_vgg16_layer_by_layer_vs_oracle():
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.vgg16().to(DEV, torch.bfloat16).to(memory_format=torch.channels_last)
    m.eval()
    for name, p in m.named_parameters():
        parts = name.split(".")
        p.requires_grad_(name.startswith("classifier.") or int(parts[1]) >= 17
                         if parts[0] == "features" else True)
    gen = torch.Generator(device=DEV).manual_seed(2)
    x = torch.randn((2, 3, 64, 64), generator=gen, device=DEV).to(torch.bfloat16)
    x = x.contiguous(memory_format=torch.channels_last)
    n = _layer_by_layer(m, x, "vgg16")
    assert n >= 30, n


FIG1_SHAPES = [(2, 8, 20, 36), (1, 8, 9, 260), (3, 8, 64, 128), (32, 8, 256, 256)]


@pytest.mark.parametrize("shape", FIG1_SHAPES)
def test_fig1_conv_3xtf32_tensor_cores(shape):
    """The Fig. 1 conv (8 -> 8, 3x3/1/1, fp32 NCHW) runs fwd and dX on the tcgen05
    kind::tf32 kernel (3xTF32 split) and dW on the CUDA-core partial-sum kernel;
    all three at the fp32 bar (rtol 1e-5 vs the f64 oracle)."""
    n, c, h, w = shape
    gen = torch.Generator(device=DEV).manual_seed(n * h + w)
    x = torch.randn(shape, generator=gen, device=DEV).requires_grad_(True)
    wt = (torch.randn((8, 8, 3, 3), generator=gen, device=DEV) / 24).requires_grad_(True)
    g = torch.randn(shape, generator=gen, device=DEV)
    u0 = launch_stats()["umma"]
    y = MF.conv2d(x, wt, None, 1, 1)
    y.backward(g)
    torch.cuda.synchronize()
    assert launch_stats()["umma"] - u0 >= 2  # fwd and dX on the tensor cores
    k = min(n, 2)
    xq, gq, wq = _np(x), _np(g), _np(wt)
    oracle.assert_close_fp32(_np(y[:k]), oracle.conv2d_fwd(xq[:k], wq, 1, 1), what="y")
    oracle.assert_close_fp32(_np(x.grad[:k]), oracle.conv2d_dx(gq[:k], wq, 1, 1, h, w),
                             what="dx")
    oracle.assert_close_fp32(_np(wt.grad), oracle.conv2d_dw(xq, gq, 1, 1, 3, 3), what="dW")
