"""Drop-in modules: ``MemSaveLinear``, ``MemSaveConv2d``, ``MemSaveBatchNorm2d``
and the module swap ``convert_to_memory_saving`` (the ``memsave_torch.nn`` API
named by the north star; the paper describes it at PAPER.md:244-253, the
reference specifies the swap as ``convert_network``).

Each ``MemSave*`` class subclasses its ``torch.nn`` counterpart, keeps the same
constructor arguments, parameters, buffers and state_dict keys, and only
replaces ``forward`` with the selective-save function from
:mod:`paper_2404_12406_b200.functional`.
"""

from __future__ import annotations

import operator

import torch
from torch import nn

from .. import functional as MF

__all__ = ["MemSaveLinear", "MemSaveConv2d", "MemSaveBatchNorm2d", "MemSaveReLU",
           "MemSaveMaxPool2d", "MemSaveDropout", "MemSaveLayerNorm", "MemSaveConvTranspose2d",
           "convert_to_memory_saving", "fuse_conv_bn_relu", "fuse_linear_gelu",
           "fuse_linear_dropout_add"]


def _share_params(dst: nn.Module, src: nn.Module, clone: bool) -> None:
    for name, p in src.named_parameters(recurse=False):
        if clone:
            p = nn.Parameter(p.detach().clone(), requires_grad=p.requires_grad)
        setattr(dst, name, p)
    for name, b in src.named_buffers(recurse=False):
        if b is not None and clone:
            b = b.clone()
        dst.register_buffer(name, b, persistent=name not in src._non_persistent_buffers_set)
    dst.train(src.training)


class MemSaveLinear(nn.Linear):
    """nn.Linear whose autograd keeps X only if W needs a grad and W only if X
    needs a grad (identical to stock torch for Linear, PAPER.md:609 / SPEC.md:248)."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return MF.linear(x, self.weight, self.bias)

    @classmethod
    def from_nn_Linear(cls, linear: nn.Linear, clone_params: bool = False) -> "MemSaveLinear":
        m = cls(linear.in_features, linear.out_features, bias=linear.bias is not None,
                device="meta", dtype=linear.weight.dtype)
        _share_params(m, linear, clone_params)
        return m


def _numeric_padding(conv: nn.Conv2d):
    p = conv.padding
    if isinstance(p, str):
        if p == "valid":
            return (0, 0)
        # 'same' (stride 1): symmetric only
        pads = []
        for k, d in zip(conv.kernel_size, conv.dilation):
            tot = d * (k - 1)
            if tot % 2:
                raise NotImplementedError("MemSaveConv2d: asymmetric 'same' padding is unsupported")
            pads.append(tot // 2)
        return tuple(pads)
    return tuple(p)


def conv2d_supported(conv: nn.Conv2d) -> bool:
    """Variants the kernels implement: groups=1, dilation=1, zero padding mode."""
    try:
        _numeric_padding(conv)
    except NotImplementedError:
        return False
    return (conv.groups == 1 and tuple(conv.dilation) == (1, 1)
            and conv.padding_mode == "zeros" and type(conv).__name__ in ("Conv2d", "MemSaveConv2d"))


class MemSaveConv2d(nn.Conv2d):
    """nn.Conv2d that saves the input only if the weight needs a gradient and the
    weight only if the input needs one (rules.py:68-71, MEMSAVE row)."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not conv2d_supported(self):
            raise NotImplementedError("MemSaveConv2d supports groups=1, dilation=1, "
                                      "padding_mode='zeros' only")
        return MF.conv2d(x, self.weight, self.bias, self.stride, _numeric_padding(self))

    @classmethod
    def from_nn_Conv2d(cls, conv: nn.Conv2d, clone_params: bool = False) -> "MemSaveConv2d":
        m = cls(conv.in_channels, conv.out_channels, conv.kernel_size, stride=conv.stride,
                padding=conv.padding, dilation=conv.dilation, groups=conv.groups,
                bias=conv.bias is not None, padding_mode=conv.padding_mode, device="meta",
                dtype=conv.weight.dtype)
        _share_params(m, conv, clone_params)
        return m


class MemSaveBatchNorm2d(nn.BatchNorm2d):
    """nn.BatchNorm2d that, in eval mode, saves the input only if the weight needs
    a gradient (rules.py:84-87, MEMSAVE row).  Training mode has
    the same storage under both policies (rules.py:74-83) and runs the stock op."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if self.training or not self.track_running_stats or self.running_mean is None:
            return super().forward(x)
        return MF.batch_norm_eval(x, self.running_mean, self.running_var, self.weight, self.bias,
                                  self.eps)

    @classmethod
    def from_nn_BatchNorm2d(cls, bn: nn.BatchNorm2d,
                            clone_params: bool = False) -> "MemSaveBatchNorm2d":
        m = cls(bn.num_features, eps=bn.eps, momentum=bn.momentum, affine=bn.affine,
                track_running_stats=bn.track_running_stats, device="meta",
                dtype=(bn.weight.dtype if bn.weight is not None else None))
        _share_params(m, bn, clone_params)
        return m


class MemSaveReLU(nn.ReLU):
    """nn.ReLU that keeps a 1-bit mask of x > 0 for backward instead of its output
    (rules.py:98-101, MEMSAVE row; saved.py:53-71)."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return MF.relu(x, self.inplace)

    @classmethod
    def from_nn_ReLU(cls, relu: nn.ReLU) -> "MemSaveReLU":
        m = cls(inplace=relu.inplace)
        m.train(relu.training)
        return m


def maxpool2d_supported(mp: nn.MaxPool2d) -> bool:
    d = mp.dilation if isinstance(mp.dilation, tuple) else (mp.dilation, mp.dilation)
    return (not mp.ceil_mode and not mp.return_indices and tuple(d) == (1, 1)
            and type(mp).__name__ in ("MaxPool2d", "MemSaveMaxPool2d"))


class MemSaveMaxPool2d(nn.MaxPool2d):
    """nn.MaxPool2d that keeps a 1-byte window argmax for backward instead of an
    int64 index tensor (rules.py:108-109; saved.py:111-125)."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not maxpool2d_supported(self):
            raise NotImplementedError("MemSaveMaxPool2d supports dilation=1, ceil_mode=False, "
                                      "return_indices=False only")
        return MF.max_pool2d(x, self.kernel_size, self.stride, self.padding)

    @classmethod
    def from_nn_MaxPool2d(cls, mp: nn.MaxPool2d) -> "MemSaveMaxPool2d":
        m = cls(mp.kernel_size, stride=mp.stride, padding=mp.padding, dilation=mp.dilation,
                return_indices=mp.return_indices, ceil_mode=mp.ceil_mode)
        m.train(mp.training)
        return m


class MemSaveDropout(nn.Dropout):
    """nn.Dropout that keeps only its 16-byte RNG key for backward and replays
    the mask (rules.py:103-106, MEMSAVE row; saved.py:91-108).  Each call draws
    a fresh seed from torch's default CPU generator; the stream is
    ``DROPOUT_STREAM_BASE + node`` (core.py:104-108).  ``generator``:
    "philox4x32" (default) or "reference" (the reference's Philox4x64 masks)."""

    def __init__(self, p: float = 0.5, inplace: bool = False, node: int = 0,
                 generator: str = "philox4x32"):
        super().__init__(p, inplace)
        self.node = int(node)
        self.generator = generator

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return MF.dropout(x, self.p, self.training, self.inplace,
                          stream=MF.DROPOUT_STREAM_BASE + self.node, generator=self.generator)

    @classmethod
    def from_nn_Dropout(cls, do: nn.Dropout, node: int = 0) -> "MemSaveDropout":
        m = cls(do.p, do.inplace, node)
        m.train(do.training)
        return m


class MemSaveLayerNorm(nn.LayerNorm):
    """nn.LayerNorm on the sm_100a kernels.  Its storage rule is the same under
    both policies (rules.py:89-96: x + per-row stats iff x or w needs a grad, w
    iff x does); db reads nothing."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return MF.layer_norm(x, self.normalized_shape, self.weight, self.bias, self.eps)

    @classmethod
    def from_nn_LayerNorm(cls, ln: nn.LayerNorm, clone_params: bool = False) -> "MemSaveLayerNorm":
        kw = {}
        if "bias" in nn.LayerNorm.__init__.__code__.co_varnames:
            kw["bias"] = ln.bias is not None
        m = cls(ln.normalized_shape, eps=ln.eps, elementwise_affine=ln.elementwise_affine,
                device="meta", dtype=(ln.weight.dtype if ln.weight is not None else None), **kw)
        _share_params(m, ln, clone_params)
        return m


def conv_transpose2d_supported(ct: nn.ConvTranspose2d) -> bool:
    d = ct.dilation if isinstance(ct.dilation, tuple) else (ct.dilation, ct.dilation)
    return (ct.groups == 1 and tuple(d) == (1, 1) and ct.padding_mode == "zeros"
            and not isinstance(ct.padding, str))


class MemSaveConvTranspose2d(nn.ConvTranspose2d):
    """nn.ConvTranspose2d with the linear-family storage rule (rules.py:68-71,
    MEMSAVE): X only if W needs a grad, W only if X needs one."""

    def forward(self, x: torch.Tensor, output_size=None) -> torch.Tensor:
        if not conv_transpose2d_supported(self):
            raise NotImplementedError("MemSaveConvTranspose2d supports groups=1, dilation=1, "
                                      "zeros padding only")
        opad = self._output_padding(x, output_size, self.stride, self.padding, self.kernel_size,
                                    2, self.dilation)
        return MF.conv_transpose2d(x, self.weight, self.bias, self.stride, self.padding, opad)

    @classmethod
    def from_nn_ConvTranspose2d(cls, ct: nn.ConvTranspose2d,
                                clone_params: bool = False) -> "MemSaveConvTranspose2d":
        m = cls(ct.in_channels, ct.out_channels, ct.kernel_size, stride=ct.stride,
                padding=ct.padding, output_padding=ct.output_padding, groups=ct.groups,
                bias=ct.bias is not None, dilation=ct.dilation, padding_mode=ct.padding_mode,
                device="meta", dtype=ct.weight.dtype)
        _share_params(m, ct, clone_params)
        return m


_MEMSAVE_TYPES = (MemSaveLinear, MemSaveConv2d, MemSaveBatchNorm2d, MemSaveReLU,
                  MemSaveMaxPool2d, MemSaveDropout, MemSaveLayerNorm, MemSaveConvTranspose2d)


def _convert_one(mod: nn.Module, kinds: dict, clone_params: bool, counter: list):
    if isinstance(mod, _MEMSAVE_TYPES):
        return None  # idempotent
    if kinds.get("dropout") and type(mod) is nn.Dropout:
        counter[0] += 1
        return MemSaveDropout.from_nn_Dropout(mod, node=counter[0] - 1)
    if kinds.get("layernorm") and type(mod) is nn.LayerNorm:
        return MemSaveLayerNorm.from_nn_LayerNorm(mod, clone_params)
    if (kinds.get("conv_transpose2d") and type(mod) is nn.ConvTranspose2d
            and conv_transpose2d_supported(mod)):
        return MemSaveConvTranspose2d.from_nn_ConvTranspose2d(mod, clone_params)
    if kinds.get("linear") and type(mod) is nn.Linear:
        return MemSaveLinear.from_nn_Linear(mod, clone_params)
    if kinds.get("conv2d") and type(mod) is nn.Conv2d and conv2d_supported(mod):
        return MemSaveConv2d.from_nn_Conv2d(mod, clone_params)
    if kinds.get("batchnorm2d") and type(mod) is nn.BatchNorm2d:
        return MemSaveBatchNorm2d.from_nn_BatchNorm2d(mod, clone_params)
    if kinds.get("relu") and type(mod) is nn.ReLU:
        return MemSaveReLU.from_nn_ReLU(mod)
    if kinds.get("maxpool2d") and type(mod) is nn.MaxPool2d and maxpool2d_supported(mod):
        return MemSaveMaxPool2d.from_nn_MaxPool2d(mod)
    return None


def _is_relu(node, modules) -> bool:
    if node.op == "call_module":
        return isinstance(modules.get(node.target), nn.ReLU)
    if node.op == "call_function":
        return node.target in (torch.relu, torch.nn.functional.relu, torch.relu_)
    if node.op == "call_method":
        return node.target in ("relu", "relu_")
    return False


def _is_add(node) -> bool:
    if node.op == "call_function" and node.target in (operator.add, operator.iadd, torch.add):
        return len(node.args) == 2 and not node.kwargs
    if node.op == "call_method" and node.target in ("add", "add_"):
        return len(node.args) == 2 and not node.kwargs
    return False


def fuse_conv_bn_relu(model: nn.Module, verbose: bool = False,
                      kinds: dict | None = None) -> nn.Module:
    """Graph pass (torch.fx) that fuses, without changing parameters, buffers or
    state_dict keys:

    * ``conv -> BatchNorm2d [-> ReLU]`` into one call of
      :func:`functional.conv_bn_relu` (BN affine + ReLU in the conv's tcgen05
      epilogue when the BN is in eval mode with frozen parameters; the three
      layers otherwise, decided at run time);
    * ``a + b -> ReLU`` (the residual join of a ResNet block) into
      :func:`functional.add_relu`, and ``conv -> BN -> add -> ReLU`` into
      :func:`functional.conv_bn_add_relu` (residual read in the conv epilogue);
    * ``conv -> ReLU`` (VGG) into :func:`functional.conv_relu`.

    Each intermediate is consumed only by the next op of the chain.  The saved
    set is the union of the fused layers' storage rules.  Models that torch.fx
    cannot trace are returned unchanged.

    ``kinds`` (the converter's kind filter, e.g. ``{"conv2d": False}``): a chain
    is fused only if every layer in it is of an enabled kind, so a disabled
    kind keeps its stock module and its stock storage."""
    import torch.fx as fx

    kinds = {} if kinds is None else kinds
    conv_types = (nn.Conv2d, MemSaveConv2d) if kinds.get("conv2d", True) else ()
    bn_ok = kinds.get("batchnorm2d", True)
    relu_ok = kinds.get("relu", True)

    def is_relu(node):
        return relu_ok and _is_relu(node, modules)

    class _Tracer(fx.Tracer):  # the memsave layers are leaves, like torch.nn layers
        def is_leaf_module(self, m, qualname):
            return isinstance(m, _MEMSAVE_TYPES) or super().is_leaf_module(m, qualname)

    try:
        gm = fx.GraphModule(model, _Tracer().trace(model), type(model).__name__)
    except Exception as exc:  # data-dependent control flow, unsupported ops ...
        if verbose:
            print(f"memsave: fx tracing failed ({type(exc).__name__}); no fusion")
        return model
    modules = dict(gm.named_modules())
    g = gm.graph
    nfused = nadd = 0
    for node in list(g.nodes):
        if (not bn_ok or node.op != "call_module"
                or not isinstance(modules.get(node.target), nn.BatchNorm2d)):
            continue
        src = node.args[0] if node.args else None
        if (not isinstance(src, fx.Node) or src.op != "call_module"
                or type(modules.get(src.target)) not in conv_types
                or len(src.users) != 1 or len(node.args) != 1 or node.kwargs):
            continue
        users = list(node.users)
        relu_node = users[0] if len(users) == 1 and is_relu(users[0]) else None
        last = relu_node or node
        with g.inserting_before(node):
            conv_ref = g.get_attr(src.target)
            bn_ref = g.get_attr(node.target)
            fused = g.call_function(MF.conv_bn_relu,
                                    (src.args[0], conv_ref, bn_ref, relu_node is not None))
        last.replace_all_uses_with(fused)
        for dead in ([relu_node] if relu_node else []) + [node, src]:
            g.erase_node(dead)
        nfused += 1
    for node in list(g.nodes):
        if not _is_add(node) or len(node.users) != 1:
            continue
        r = next(iter(node.users))
        if not is_relu(r):
            continue
        a, b = node.args
        if not (isinstance(a, fx.Node) and isinstance(b, fx.Node)):
            continue
        with g.inserting_before(node):
            fused = g.call_function(MF.add_relu, (a, b))
        r.replace_all_uses_with(fused)
        g.erase_node(r)
        g.erase_node(node)
        nadd += 1
    # conv -> relu without a BN (VGG): ReLU and its mask in the conv epilogue
    nrelu = 0
    for node in list(g.nodes):
        if node.op != "call_module" or type(modules.get(node.target)) not in conv_types:
            continue
        users = list(node.users)
        if len(users) != 1 or not is_relu(users[0]) or len(node.args) != 1:
            continue
        with g.inserting_before(node):
            conv_ref = g.get_attr(node.target)
            fused = g.call_function(MF.conv_relu, (node.args[0], conv_ref))
        users[0].replace_all_uses_with(fused)
        g.erase_node(users[0])
        g.erase_node(node)
        nrelu += 1
    # conv -> bn (no relu) whose only consumer is an add -> relu join: one launch
    # with the residual added in the conv epilogue
    nres = 0
    for node in list(g.nodes):
        if node.op != "call_function" or node.target is not MF.add_relu:
            continue
        a, b = node.args
        for main, other in ((a, b), (b, a)):
            if (isinstance(main, fx.Node) and main.op == "call_function"
                    and main.target is MF.conv_bn_relu and main.args[3] is False
                    and len(main.users) == 1):
                with g.inserting_before(node):
                    fused = g.call_function(MF.conv_bn_add_relu,
                                            (main.args[0], main.args[1], main.args[2], other))
                node.replace_all_uses_with(fused)
                g.erase_node(node)
                g.erase_node(main)
                nres += 1
                break
    # generic form: every fused chain becomes fused_conv(...) -> (y, mask, alias)
    gen = []
    for node in list(g.nodes):
        if node.op != "call_function" or node.target not in (MF.conv_bn_relu, MF.conv_relu,
                                                             MF.conv_bn_add_relu):
            continue
        kw = {}
        if node.target is MF.conv_bn_relu:
            x, conv_ref, bn_ref, r = node.args
        elif node.target is MF.conv_relu:
            (x, conv_ref), bn_ref, r = node.args, None, True
        else:
            x, conv_ref, bn_ref, res = node.args
            r, kw = True, {"residual": res}
        with g.inserting_before(node):
            f = g.call_function(MF.fused_conv, (x, conv_ref, bn_ref, r), kw)
            y = g.call_function(operator.getitem, (f, 0))
        node.replace_all_uses_with(y)
        g.erase_node(node)
        gen.append((f, y))
    # a tensor read as the input of a fused conv and by one more fused chain (a
    # ResNet block input: conv1 and the identity / downsample branch): the conv
    # tees it, so the two gradients are summed in its dgrad epilogue rather than
    # by a separate pass
    ntee = 0
    order = {n: i for i, n in enumerate(g.nodes)}
    for node in list(g.nodes):
        users = sorted(node.users, key=lambda n: order.get(n, len(order)))
        if len(users) != 2:
            continue
        u1, u2 = users
        if (u1.target is not MF.fused_conv or u1.args[0] is not node
                or node in u1.args[1:] or node in u1.kwargs.values()
                or u2.target is not MF.fused_conv):
            continue
        u1.kwargs = {**u1.kwargs, "tee": True}
        with g.inserting_after(u1):
            alias = g.call_function(operator.getitem, (u1, 2))
        u2.args = tuple(alias if a is node else a for a in u2.args)
        u2.kwargs = {k: (alias if v is node else v) for k, v in u2.kwargs.items()}
        ntee += 1
    # a fused ReLU whose output feeds only the input of another fused conv: that
    # conv applies the ReLU's backward (keep mask [* BN scale]) in its dgrad
    # epilogue instead of a separate pass over the gradient
    nfwd = 0
    for f, y in gen:
        if not f.args[3] or len(y.users) != 1:
            continue
        c = next(iter(y.users))
        pool = modules.get(c.target) if c.op == "call_module" else None
        is_pool = (isinstance(pool, MemSaveMaxPool2d) and maxpool2d_supported(pool)
                   and c.args == (y,) and not c.kwargs)
        if not is_pool and (c.target is not MF.fused_conv or c.args[0] is not y
                            or y in c.args[1:] or y in c.kwargs.values()):
            continue
        f.kwargs = {**f.kwargs, "raw": True}
        with g.inserting_after(y):
            m = g.call_function(operator.getitem, (f, 1))
        in_bn = f.args[2] if "residual" not in f.kwargs else None
        if is_pool:  # the stem: conv -> BN -> ReLU -> MaxPool
            with g.inserting_before(c):
                mp = g.call_function(MF.max_pool2d, (y, pool.kernel_size, pool.stride,
                                                     pool.padding),
                                     {"in_mask": m, "in_bn": in_bn})
            c.replace_all_uses_with(mp)
            g.erase_node(c)
        else:
            c.kwargs = {**c.kwargs, "in_mask": m, "in_bn": in_bn}
        nfwd += 1
    g.eliminate_dead_code()
    g.lint()
    gm.recompile()
    if verbose:
        print(f"memsave: fused {nfused} conv->bn[->relu], {nadd} add->relu, {nres} "
              f"conv->bn->add->relu and {nrelu} conv->relu chains; {ntee} tee'd inputs, "
              f"{nfwd} ReLU backwards moved into the consumer's dgrad")
    return gm


_GELU_FNS = (torch.nn.functional.gelu, torch._C._nn.gelu)


def _is_gelu(node, modules) -> bool:
    """an exact (erf) GELU: F.gelu / nn.GELU with approximate='none'"""
    if node.op == "call_module":
        m = modules.get(node.target)
        return type(m) is nn.GELU and m.approximate == "none" and len(node.args) == 1
    if node.op == "call_function" and node.target in _GELU_FNS:
        approx = node.kwargs.get("approximate", node.args[1] if len(node.args) > 1 else "none")
        return approx == "none" and set(node.kwargs) <= {"approximate"}
    return False


def _gelu_layer(x: torch.Tensor, lin: nn.Linear) -> torch.Tensor:
    return MF.linear_gelu(x, lin.weight, lin.bias)


def _simple_graph(gm, modules) -> bool:
    """only placeholders, leaf-module calls, GELU / add calls and the output: a
    module whose trace cannot have baked in a data- or argument-dependent branch"""
    for n in gm.graph.nodes:
        if n.op in ("placeholder", "output", "get_attr", "call_module"):
            continue
        if n.op == "call_function" and (n.target in _GELU_FNS or _is_add(n)):
            continue
        return False
    return True


def _rewrite_linear_gelu(gm) -> int:
    import torch.fx as fx

    modules = dict(gm.named_modules())
    g = gm.graph
    n = 0
    for node in list(g.nodes):
        if node.op != "call_module" or type(modules.get(node.target)) is not MemSaveLinear:
            continue
        users = list(node.users)
        if len(users) != 1 or len(node.args) != 1 or node.kwargs or not _is_gelu(users[0], modules):
            continue
        if not isinstance(node.args[0], fx.Node):
            continue
        with g.inserting_before(node):
            ref = g.get_attr(node.target)
            fused = g.call_function(_gelu_layer, (node.args[0], ref))
        users[0].replace_all_uses_with(fused)
        g.erase_node(users[0])
        g.erase_node(node)
        n += 1
    if n:
        g.eliminate_dead_code()
        g.lint()
        gm.recompile()
    return n


def _dropout_add_layer(x: torch.Tensor, lin: nn.Linear, drop, other: torch.Tensor):
    y_shape = tuple(x.shape[:-1]) + (lin.out_features,)
    if (tuple(other.shape) != y_shape or other.dtype != x.dtype
            or type(drop) is not MemSaveDropout or drop.inplace):
        return drop(lin(x)) + other
    return MF.linear_dropout_add(x, lin.weight, lin.bias, other, drop.p, drop.training,
                                 stream=MF.DROPOUT_STREAM_BASE + drop.node,
                                 generator=drop.generator)


def _rewrite_linear_dropout_add(gm) -> int:
    """dense -> MemSaveDropout -> add(., other) with single-use intermediates"""
    import torch.fx as fx

    modules = dict(gm.named_modules())
    g = gm.graph
    n = 0
    for node in list(g.nodes):
        if node.op != "call_module" or type(modules.get(node.target)) is not MemSaveLinear:
            continue
        if len(node.users) != 1 or len(node.args) != 1 or node.kwargs:
            continue
        d = next(iter(node.users))
        if (d.op != "call_module" or type(modules.get(d.target)) is not MemSaveDropout
                or len(d.users) != 1 or d.args != (node,) or d.kwargs):
            continue
        a = next(iter(d.users))
        if not _is_add(a) or a.op != "call_function":
            continue
        other = a.args[1] if a.args[0] is d else a.args[0]
        if other is d or not isinstance(other, fx.Node) or not isinstance(node.args[0], fx.Node):
            continue
        with g.inserting_before(a):
            lref = g.get_attr(node.target)
            dref = g.get_attr(d.target)
            fused = g.call_function(_dropout_add_layer, (node.args[0], lref, dref, other))
        a.replace_all_uses_with(fused)
        for dead in (a, d, node):
            g.erase_node(dead)
        n += 1
    if n:
        g.eliminate_dead_code()
        g.lint()
        gm.recompile()
    return n


def _fuse_per_module(model: nn.Module, rewrite, what: str, verbose: bool) -> nn.Module:
    """Runs ``rewrite`` on the traced graph of every module whose ``forward``
    takes only required arguments and traces to a plain chain of leaf layers,
    GELUs and adds (e.g. BERT's intermediate / output blocks); a rewritten
    module is replaced by its ``fx.GraphModule`` (same parameters and state_dict
    keys), any other module is searched recursively."""
    import inspect

    import torch.fx as fx

    class _Tracer(fx.Tracer):
        def is_leaf_module(self, m, qualname):
            return isinstance(m, _MEMSAVE_TYPES) or super().is_leaf_module(m, qualname)

    total = [0]

    def candidate(mod) -> bool:
        if isinstance(mod, _MEMSAVE_TYPES) or not any(
                type(c) is MemSaveLinear for c in mod.children()):
            return False
        try:
            params = inspect.signature(mod.forward).parameters.values()
        except (TypeError, ValueError):
            return False
        return all(p.default is inspect.Parameter.empty and
                   p.kind in (p.POSITIONAL_ONLY, p.POSITIONAL_OR_KEYWORD) for p in params)

    def try_mod(mod):
        if not candidate(mod):
            return None
        try:
            gm = fx.GraphModule(mod, _Tracer().trace(mod), type(mod).__name__)
        except Exception:
            return None
        if not _simple_graph(gm, dict(gm.named_modules())):
            return None
        k = rewrite(gm)
        total[0] += k
        return gm if k else None

    def walk(parent):
        for name, child in list(parent.named_children()):
            new = try_mod(child)
            if new is not None:
                new.train(child.training)
                setattr(parent, name, new)
            else:
                walk(child)

    top = try_mod(model)
    if top is None:
        walk(model)
    if verbose:
        print(f"memsave: fused {total[0]} {what}")
    return top if top is not None else model


def fuse_linear_gelu(model: nn.Module, verbose: bool = False) -> nn.Module:
    """Fuses ``MemSaveLinear -> GELU(erf)`` into one :func:`functional.linear_gelu`
    node (GELU in the GEMM epilogue, pre-activation and output from one pass).
    Opt-in: at BERT's FFN shape (32768 x 3072 x 768) the fused launch takes
    285 us against 136 us + 112 us for the GEMM and torch's GELU -- the erf's
    ~17 instructions per element in the 8 epilogue warps outlast the MMAs.
    Works per module (:func:`_fuse_per_module`); returns the model (or its
    replacement when the root itself was rewritten)."""
    return _fuse_per_module(model, _rewrite_linear_gelu, "linear->gelu pairs", verbose)


def fuse_linear_dropout_add(model: nn.Module, verbose: bool = False) -> nn.Module:
    """Fuses ``MemSaveLinear -> MemSaveDropout -> + residual`` (a transformer
    block's output projection) into one :func:`functional.linear_dropout_add`
    node: dropout and residual add in the GEMM epilogue, values and saved set
    equal to the three layers'.  Works per module like :func:`fuse_linear_gelu`;
    run by ``convert_to_memory_saving(fuse=True)``."""
    return _fuse_per_module(model, _rewrite_linear_dropout_add, "linear->dropout->add chains",
                            verbose)


def convert_to_memory_saving(model: nn.Module, linear: bool = True, conv2d: bool = True,
                             conv1d: bool = False, conv3d: bool = False,
                             batchnorm2d: bool = True, relu: bool = True,
                             maxpool2d: bool = True, layernorm: bool = True,
                             dropout: bool = True, conv_transpose2d: bool = True,
                             verbose: bool = False, clone_params: bool = False,
                             fuse: bool = False) -> nn.Module:
    """Swap supported layers of ``model`` for their MemSave equivalents, in place.

    Mirrors the reference ``convert_network(net, target, layer_filter)``
    (SPEC.md:320-328): the boolean flags are the kind filter, conversion is
    idempotent, parameters are shared with the original modules unless
    ``clone_params``.  The SURVEY.md §8(f) rows ReLU (bit mask), MaxPool2d
    (1-byte argmax), Dropout (RNG replay; node i of the traversal draws from
    stream DROPOUT_STREAM_BASE + i), LayerNorm and ConvTranspose2d are swapped
    too; conv1d/3d are accepted for API compatibility and left untouched.
    ``fuse=True`` additionally runs :func:`fuse_linear_dropout_add` (per
    module) and :func:`fuse_conv_bn_relu` (returns an ``fx.GraphModule``
    sharing the parameters, or the model unchanged when it cannot be traced).  :func:`fuse_linear_gelu` is opt-in (measured slower
    than the two launches on B200 at the BERT FFN shape).
    Returns the (possibly replaced) model.
    """
    kinds = {"linear": linear, "conv2d": conv2d, "batchnorm2d": batchnorm2d, "relu": relu,
             "maxpool2d": maxpool2d, "layernorm": layernorm, "dropout": dropout,
             "conv_transpose2d": conv_transpose2d}
    counter = [0]
    top = _convert_one(model, kinds, clone_params, counter)
    if top is not None:
        if verbose:
            print(f"memsave: {type(model).__name__} -> {type(top).__name__}")
        return top

    def walk(parent: nn.Module, prefix: str):
        for name, child in list(parent.named_children()):
            new = _convert_one(child, kinds, clone_params, counter)
            if new is not None:
                setattr(parent, name, new)
                if verbose:
                    print(f"memsave: {prefix}{name}: {type(child).__name__} -> "
                          f"{type(new).__name__}")
            else:
                walk(child, f"{prefix}{name}.")

    walk(model, "")
    if fuse:
        if linear and dropout:
            model = fuse_linear_dropout_add(model, verbose=verbose)
        return fuse_conv_bn_relu(model, verbose=verbose, kinds=kinds)
    return model
