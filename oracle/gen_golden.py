"""Generate the golden fixtures under tests/golden/ (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

* conv2d: inputs drawn with the reference's own Philox generator
  (leantape.core.Rng, core.py:100-124; stream 0 = input, 1 = weight,
  2 = upstream gradient), outputs computed by the reference kernels
  (leantape.kernels.conv2d_fwd/dx/dw, kernels/__init__.py:26-30) in float64 with
  the numba backend, cross-checked against its numpy backend.
* rules: the full storage_decision table of leantape.rules (rules.py:57-141)
  for the hot-path kinds over every flag combination.
* linear / batchnorm2d-eval: the reference has only SPEC formulas
  (SPEC.md:245, :269); vectors come from torch-CPU float64 autograd of the
  same formulas.

The reference is NOT available on the GPU box; this script only runs here and
its outputs are committed.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")

# (name, N, Cin, H, W, Cout, k, stride, pad) — config geometries at desk scale
CONV_CASES = [
    ("fig1_3x3s1p1", 2, 8, 16, 16, 8, 3, 1, 1),
    ("res_3x3s2p1", 2, 16, 13, 11, 24, 3, 2, 1),
    ("res_1x1s2p0", 2, 16, 10, 12, 32, 1, 2, 0),
    ("stem_7x7s2p3", 1, 3, 21, 19, 16, 7, 2, 3),
    ("res_1x1s1p0", 3, 24, 7, 7, 16, 1, 1, 0),
    ("odd_3x3s1p0", 2, 5, 9, 8, 6, 3, 1, 0),
    ("unit_1x1", 1, 1, 4, 5, 1, 1, 1, 0),
]


def gen_conv(core, kernels):
    out = {}
    for (name, n, cin, h, w, cout, k, s, p) in CONV_CASES:
        x = core.Rng(0, 0).normal((n, cin, h, w), core.Dtype.F64)
        wt = core.Rng(0, 1).normal((cout, cin, k, k), core.Dtype.F64)
        if name == "unit_1x1":
            wt = np.ones_like(wt)
        y = kernels.conv2d_fwd(x, wt, s, p)
        g = core.Rng(0, 2).normal(y.shape, core.Dtype.F64)
        dx = kernels.conv2d_dx(g, wt, s, p, h, w)
        dw = kernels.conv2d_dw(x, g, s, p, k, k)
        for key, val in dict(x=x, w=wt, y=y, g=g, dx=dx, dw=dw).items():
            out[f"{name}/{key}"] = np.ascontiguousarray(val)
        out[f"{name}/geom"] = np.array([n, cin, h, w, cout, k, s, p], dtype=np.int64)
    return out


POOL_CASES = [
    # name, shape, kh, kw, sh, sw
    ("mp_2x2s2", (2, 3, 8, 6), 2, 2, 2, 2),
    ("mp_3x3s2", (2, 4, 9, 11), 3, 3, 2, 2),
    ("mp_3x3s1", (1, 2, 7, 5), 3, 3, 1, 1),
    ("mp_ties", (1, 2, 6, 6), 3, 3, 2, 2),
]


def gen_pool(core, kernels):
    out = {}
    for name, shape, kh, kw, sh, sw in POOL_CASES:
        x = core.Rng(3, 0).normal(shape, core.Dtype.F64)
        if name == "mp_ties":
            x = np.round(x)  # many ties: checks the first-occurrence rule
        y, idx = kernels.maxpool2d_fwd(x, kh, kw, sh, sw)
        g = core.Rng(3, 2).normal(y.shape, core.Dtype.F64)
        dx = kernels.maxpool2d_bwd(g, idx, shape[2], shape[3])
        for key, val in dict(x=x, y=y, idx=idx, g=g, dx=dx).items():
            out[f"{name}/{key}"] = np.ascontiguousarray(val)
        out[f"{name}/geom"] = np.array([kh, kw, sh, sw], dtype=np.int64)
    return out


def gen_rules(rules):
    table = []
    for kind in ("linear", "conv2d", "conv_transpose2d", "batchnorm2d", "relu", "maxpool2d",
                 "dropout", "layernorm"):
        for bn_train in ((False, True) if kind == "batchnorm2d" else (False,)):
            for pol in (rules.Policy.NAIVE, rules.Policy.MEMSAVE):
                for x_rg in (False, True):
                    for w_rg in (False, True):
                        for b_rg in (False, True):
                            out_rg = x_rg or w_rg or b_rg
                            saves = rules.storage_decision(kind, pol, x_rg=x_rg, w_rg=w_rg,
                                                           out_rg=out_rg, bn_train=bn_train)
                            table.append(dict(kind=kind, bn_train=bn_train, policy=pol.value,
                                              x_rg=x_rg, w_rg=w_rg, b_rg=b_rg,
                                              out_rg=out_rg, saves=[list(t) for t in saves]))
    return table


def gen_linear_bn(core):
    import torch
    out = {}
    # Linear
    for name, lead, fin, fout in (("lin_small", (3,), 4, 5), ("lin_3d", (2, 7), 16, 24)):
        x = core.Rng(1, 0).normal(lead + (fin,), core.Dtype.F64)
        w = core.Rng(1, 1).normal((fout, fin), core.Dtype.F64)
        b = core.Rng(1, 3).normal((fout,), core.Dtype.F64)
        tx, tw, tb = (torch.tensor(a, requires_grad=True) for a in (x, w, b))
        y = torch.nn.functional.linear(tx, tw, tb)
        g = core.Rng(1, 2).normal(tuple(y.shape), core.Dtype.F64)
        y.backward(torch.tensor(g))
        for key, val in dict(x=x, w=w, b=b, y=y.detach().numpy(), g=g, dx=tx.grad.numpy(),
                             dw=tw.grad.numpy(), db=tb.grad.numpy()).items():
            out[f"{name}/{key}"] = np.ascontiguousarray(val)
    # BatchNorm2d eval
    for name, shape in (("bn_small", (2, 3, 4, 5)), ("bn_odd", (3, 7, 5, 3))):
        c = shape[1]
        x = core.Rng(2, 0).normal(shape, core.Dtype.F64)
        w = core.Rng(2, 1).normal((c,), core.Dtype.F64)
        b = core.Rng(2, 3).normal((c,), core.Dtype.F64)
        mean = 0.1 * core.Rng(2, 4).normal((c,), core.Dtype.F64)
        var = 0.5 + 1.5 * core.Rng(2, 5).uniform((c,))
        eps = 1e-5
        tx, tw, tb = (torch.tensor(a, requires_grad=True) for a in (x, w, b))
        y = torch.nn.functional.batch_norm(tx, torch.tensor(mean), torch.tensor(var), tw, tb,
                                           training=False, eps=eps)
        g = core.Rng(2, 2).normal(shape, core.Dtype.F64)
        y.backward(torch.tensor(g))
        for key, val in dict(x=x, w=w, b=b, mean=mean, var=var, y=y.detach().numpy(), g=g,
                             dx=tx.grad.numpy(), dw=tw.grad.numpy(),
                             db=tb.grad.numpy()).items():
            out[f"{name}/{key}"] = np.ascontiguousarray(val)
        out[f"{name}/eps"] = np.array(eps)
    return out


def gen_dropout(core):
    """Dropout keep masks from the reference generator: Rng(seed, stream).uniform
    (core.py:100-124) >= p, for streams DROPOUT_STREAM_BASE + node."""
    out = {}
    base = core.Rng.DROPOUT_STREAM_BASE
    for name, seed, node, p, n in (("d_small", 0, 0, 0.1, 37), ("d_half", 12345, 3, 0.5, 1000),
                                   ("d_big", 2 ** 61 + 7, 11, 0.25, 4099)):
        u = core.Rng(seed, base + node).uniform((n,))
        out[f"{name}/key"] = np.array([seed, base + node], dtype=np.uint64)
        out[f"{name}/p"] = np.array(p)
        out[f"{name}/mask"] = (u >= p).astype(np.uint8)
    return out


def gen_layernorm(core):
    """LayerNorm (SPEC.md forward_layernorm): torch-CPU float64 autograd."""
    import torch
    out = {}
    for name, shape, d in (("ln_small", (3, 8), 8), ("ln_3d", (2, 5, 24), 24)):
        x = core.Rng(3, 0).normal(shape, core.Dtype.F64)
        w = core.Rng(3, 1).normal((d,), core.Dtype.F64)
        b = core.Rng(3, 3).normal((d,), core.Dtype.F64)
        tx, tw, tb = (torch.tensor(a, requires_grad=True) for a in (x, w, b))
        y = torch.nn.functional.layer_norm(tx, (d,), tw, tb, eps=1e-5)
        g = core.Rng(3, 2).normal(shape, core.Dtype.F64)
        y.backward(torch.tensor(g))
        for key, val in dict(x=x, w=w, b=b, y=y.detach().numpy(), g=g, dx=tx.grad.numpy(),
                             dw=tw.grad.numpy(), db=tb.grad.numpy()).items():
            out[f"{name}/{key}"] = np.ascontiguousarray(val)
    return out


def gen_conv_transpose(core, kernels):
    """ConvTranspose2d through the reference conv kernels (SPEC.md: convT forward
    = conv2d input-VJP with the same kernel)."""
    out = {}
    for name, n, cin, h, w, cout, k, s, p in (("ct_s2", 2, 6, 5, 4, 4, 3, 2, 1),
                                              ("ct_s1", 1, 3, 6, 6, 5, 3, 1, 1)):
        x = core.Rng(4, 0).normal((n, cin, h, w), core.Dtype.F64)
        wt = core.Rng(4, 1).normal((cin, cout, k, k), core.Dtype.F64)
        ho, wo = (h - 1) * s - 2 * p + k, (w - 1) * s - 2 * p + k
        y = kernels.conv2d_dx(x, wt, s, p, ho, wo)
        g = core.Rng(4, 2).normal((n, cout, ho, wo), core.Dtype.F64)
        dx = kernels.conv2d_fwd(g, wt, s, p)
        dw = kernels.conv2d_dw(g, x, s, p, k, k)
        for key, val in dict(x=x, w=wt, y=y, g=g, dx=dx, dw=dw).items():
            out[f"{name}/{key}"] = np.ascontiguousarray(val)
        out[f"{name}/geom"] = np.array([s, p], dtype=np.int64)
    return out


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from leantape import core, rules  # noqa: E402
    from leantape import kernels  # noqa: E402
    from leantape.kernels import numpy_impl  # noqa: E402
    assert kernels.backend_name() in ("numba", "numpy")
    os.makedirs(GOLDEN, exist_ok=True)

    conv = gen_conv(core, kernels)
    # cross-check the reference's two backends against each other
    for (name, *_r) in CONV_CASES:
        n, cin, h, w, cout, k, s, p = conv[f"{name}/geom"]
        y2 = numpy_impl.conv2d_fwd(conv[f"{name}/x"], conv[f"{name}/w"], int(s), int(p))
        assert np.allclose(y2, conv[f"{name}/y"], rtol=1e-12, atol=1e-12), name
    np.savez_compressed(os.path.join(GOLDEN, "conv2d_ref.npz"), **conv)

    with open(os.path.join(GOLDEN, "rules.json"), "w") as f:
        json.dump({"source": "leantape.rules.storage_decision (rules.py:57-141)",
                   "table": gen_rules(rules)}, f, indent=1)

    np.savez_compressed(os.path.join(GOLDEN, "linear_bn_spec.npz"), **gen_linear_bn(core))
    np.savez_compressed(os.path.join(GOLDEN, "maxpool_ref.npz"), **gen_pool(core, kernels))
    np.savez_compressed(os.path.join(GOLDEN, "dropout_ref.npz"), **gen_dropout(core))
    np.savez_compressed(os.path.join(GOLDEN, "layernorm_spec.npz"), **gen_layernorm(core))
    np.savez_compressed(os.path.join(GOLDEN, "conv_transpose_ref.npz"),
                        **gen_conv_transpose(core, kernels))

    # SPEC known-answer examples
    kat = {
        "byte_size_fig1_f32": int(core.shape_bytes((256, 8, 256, 256), core.Dtype.F32)),
        "byte_size_desk_f32": int(core.shape_bytes((4, 8, 32, 32), core.Dtype.F32)),
        "conv_backend": kernels.backend_name(),
    }
    with open(os.path.join(GOLDEN, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()
