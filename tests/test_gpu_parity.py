"""GPU parity: the sm_100a kernels (through the C ABI, via the autograd
functions) against the float64 oracle on the same quantised inputs.

Tolerances (oracle/tolerance.py):
  float32 — norm-wise rel ≤ 1e-5 and elementwise rtol 1e-5 (+1e-5·max|ref|)
  bf16    — ≤ 1 bf16 ulp (+1 % max|ref| floor) of the rounded f64 oracle and
            norm-wise rel ≤ 1e-3
"""

import numpy as np
import pytest
import torch

import oracle
from mscases import CONV_CASES
from paper_2404_12406_b200 import functional as MF
from paper_2404_12406_b200 import launch_count, launch_stats

pytestmark = pytest.mark.gpu

DEV = "cuda"
TDT = {"bf16": torch.bfloat16, "f32": torch.float32, "fp16": torch.float16}


def _close(a: torch.Tensor, ref64, dt, what, ulps=1.01):
    a = a.detach().float().cpu().double().numpy()
    if dt == "f32":
        oracle.assert_close_fp32(a, ref64, what=what)
    else:
        oracle.assert_close_lowp(a, ref64, dt, ulps=ulps, what=what)


def _q(arr, dt):
    """numpy f64 -> (torch tensor on GPU in dt, the quantised f64 values)."""
    t = torch.tensor(np.asarray(arr), dtype=torch.float64).to(TDT[dt])
    return t.to(DEV), t.double().numpy()


# ------------------------------------------------------------------ conv2d
def _conv_check(x64, w64, g64, stride, pad, dt, channels_last, with_bias=False, rg=(1, 1, 1),
                tag=""):
    x, xq = _q(x64, dt)
    w, wq = _q(w64, dt)
    g, gq = _q(g64, dt)
    b = bq = None
    if with_bias:
        b, bq = _q(np.linspace(-1, 1, w64.shape[0]), dt)
    if channels_last:
        x = x.contiguous(memory_format=torch.channels_last)
        w = w.contiguous(memory_format=torch.channels_last)
    x.requires_grad_(bool(rg[0]))
    w.requires_grad_(bool(rg[1]))
    if b is not None:
        b.requires_grad_(bool(rg[2]))
    n0 = launch_count()
    y = MF.conv2d(x, w, b, stride, pad)
    y_ref = oracle.conv2d_fwd(xq, wq, stride, pad)
    if with_bias:
        y_ref = y_ref + bq[None, :, None, None]
    _close(y, y_ref, dt, f"{tag} y")
    if any(rg):
        y.backward(g.contiguous(memory_format=torch.channels_last) if channels_last else g)
    assert launch_count() > n0  # the native library ran
    h, wd = x64.shape[2:]
    if rg[0]:
        _close(x.grad, oracle.conv2d_dx(gq, wq, stride, pad, h, wd), dt, f"{tag} dx")
    if rg[1]:
        _close(w.grad, oracle.conv2d_dw(xq, gq, stride, pad, w64.shape[2], w64.shape[3]), dt,
               f"{tag} dw")
    if with_bias and rg[2]:
        _close(b.grad, gq.sum(axis=(0, 2, 3)), dt, f"{tag} db")


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_conv_golden_vectors(conv_golden, case, dt):
    g = conv_golden
    n, cin, h, w, cout, k, s, p = (int(v) for v in g[f"{case}/geom"])
    if dt == "f32":
        # float32 against the reference outputs directly (inputs are exact f64 draws,
        # quantised to f32; the golden outputs were computed in f64 by the reference)
        x, xq = _q(g[f"{case}/x"], "f32")
        wt, wq = _q(g[f"{case}/w"], "f32")
        gy, gq = _q(g[f"{case}/g"], "f32")
        x.requires_grad_(True)
        wt.requires_grad_(True)
        y = MF.conv2d(x, wt, None, s, p)
        y.backward(gy)
        _close(y, oracle.conv2d_fwd(xq, wq, s, p), "f32", f"{case} y")
        _close(x.grad, oracle.conv2d_dx(gq, wq, s, p, h, w), "f32", f"{case} dx")
        _close(wt.grad, oracle.conv2d_dw(xq, gq, s, p, k, k), "f32", f"{case} dw")
        # and the quantisation-free check against the reference's own vectors
        if case == "unit_1x1":
            np.testing.assert_allclose(y.detach().cpu().double().numpy(), g[f"{case}/y"],
                                       rtol=1e-6)
    else:
        _conv_check(g[f"{case}/x"], g[f"{case}/w"], g[f"{case}/g"], s, p, dt,
                    channels_last=True, tag=case)


# tcgen05 implicit-GEMM geometries (channel counts multiple of 8, NHWC, bf16)
TC_CASES = [
    # n, c, h, w, k, r, stride, pad
    (2, 64, 14, 14, 128, 3, 1, 1),     # resnet 3x3 s1
    (2, 128, 15, 13, 64, 3, 2, 1),     # 3x3 s2, odd sizes (dgrad phases with unequal extents)
    (2, 64, 16, 16, 256, 1, 2, 0),     # 1x1 s2 downsample (phases without taps)
    (3, 256, 7, 7, 512, 3, 1, 1),      # layer4-like, multiple N tiles
    (2, 3, 32, 32, 64, 7, 2, 3),       # stem: 3 channels (padded activation copy)
    (2, 32, 9, 9, 40, 3, 1, 1),        # C=32 (channel OOB fill), K=40 (N tail)
    (1, 64, 10, 10, 64, 3, 1, 0),      # no padding
    (2, 16, 12, 12, 24, 5, 1, 2),      # 5x5
    (3, 3, 45, 37, 64, 7, 2, 3),       # stem, odd sizes: C8 fprop + scatter dgrad
    (2, 8, 20, 20, 32, 3, 1, 1),       # C=8: C8 fprop, 8-channel dgrad phases
    (2, 64, 9, 13, 64, 3, 1, 1),       # 64->64 3x3/1/1: halo kernel, odd H (partial tile)
    (1, 64, 56, 56, 64, 3, 1, 1),      # ResNet layer1 geometry
    (3, 64, 7, 62, 64, 3, 1, 1),       # widest row the 64-pixel pitch allows
    (1, 64, 5, 224, 64, 3, 1, 1),      # VGG conv1_2 rows: wide halo tiles, 2 x 128-px segments
    (2, 64, 3, 130, 64, 3, 1, 1),      # wide halo: a 2-pixel last segment
    (2, 3, 20, 150, 64, 3, 1, 1),      # VGG conv1_1-like: 8-ch row segments, 2 segments/row
    (1, 5, 9, 33, 32, 3, 1, 1),        # 5 channels, one partial segment
]


@pytest.mark.parametrize("case", TC_CASES)
def test_conv_tcgen05_bf16(case):
    n, c, h, w, k, r, s, p = case
    rng = np.random.default_rng(hash(case) % 2**32)
    oh = (h + 2 * p - r) // s + 1
    ow = (w + 2 * p - r) // s + 1
    x = rng.standard_normal((n, c, h, w))
    wt = rng.standard_normal((k, c, r, r)) / np.sqrt(c * r * r)
    g = rng.standard_normal((n, k, oh, ow))
    u0 = launch_stats()["umma"]
    _conv_check(x, wt, g, s, p, "bf16", channels_last=True, with_bias=True, tag=str(case))
    used = launch_stats()["umma"] - u0
    # fwd + dx always run on tcgen05; dw too when both channel counts are multiples of 8
    assert used >= (3 if c % 8 == 0 else 2), used


def test_stem_full_width():
    # ResNet stem geometry at batch 2 (224x224): many scatter tiles overlapping
    rng = np.random.default_rng(11)
    x = rng.standard_normal((2, 3, 224, 224))
    wt = rng.standard_normal((64, 3, 7, 7)) / 12
    g = rng.standard_normal((2, 64, 112, 112))
    _conv_check(x, wt, g, 2, 3, "bf16", channels_last=True, rg=(1, 0, 0), tag="stem224")


def test_conv_tcgen05_many_tiles():
    # > 148 tiles per launch: exercises the persistent tile loop and the TMEM
    # double buffer (epilogue of tile i overlapping the main loop of tile i+1)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((8, 64, 56, 56))
    wt = rng.standard_normal((64, 64, 3, 3)) / 24
    g = rng.standard_normal((8, 64, 56, 56))
    _conv_check(x, wt, g, 1, 1, "bf16", channels_last=True, rg=(1, 1, 0), tag="many")


@pytest.mark.parametrize("rg", [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)])
def test_conv_selective_products(rg):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 64, 8, 8))
    wt = rng.standard_normal((64, 64, 3, 3)) / 24
    g = rng.standard_normal((2, 64, 8, 8))
    _conv_check(x, wt, g, 1, 1, "bf16", channels_last=True, with_bias=True, rg=rg, tag=str(rg))


def test_conv_nchw_bf16_and_fp16():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 16, 9, 9))
    wt = rng.standard_normal((24, 16, 3, 3)) / 12
    g = rng.standard_normal((2, 24, 5, 5))
    _conv_check(x, wt, g, 2, 1, "bf16", channels_last=False, tag="nchw-bf16")
    _conv_check(x, wt, g, 2, 1, "fp16", channels_last=True, tag="fp16")


# ------------------------------------------------------------------ linear
LIN_CASES = [
    # lead dims, in, out
    ((4, 96), 768, 768),      # BERT-like, M=384
    ((300,), 512, 1000),      # fc with N tail
    ((2, 70), 256, 64),       # M tail
    ((8,), 4096, 256),        # tiny M, long K (split-K)
    ((513,), 64, 8),          # N = 8
    ((2, 1024), 1024, 1536),  # CTA-pair tiles (M=256 MMA), several tiles per CTA
    ((1, 640), 384, 320),     # pair with a partial second M tile, N tail of a BN=64 pair
    ((2, 1280), 1024, 2048),  # fwd: 80 pair tiles > 74 slots -> last wave K-split (tail)
    ((2, 1280), 2048, 1024),  # dX: the same for the input-VJP (MN-major B)
]


@pytest.mark.parametrize("case", LIN_CASES)
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_linear(case, dt):
    lead, fin, fout = case
    rng = np.random.default_rng(fin + fout)
    x, xq = _q(rng.standard_normal(lead + (fin,)), dt)
    w, wq = _q(rng.standard_normal((fout, fin)) / np.sqrt(fin), dt)
    b, bq = _q(rng.standard_normal(fout), dt)
    g, gq = _q(rng.standard_normal(lead + (fout,)), dt)
    for t in (x, w, b):
        t.requires_grad_(True)
    u0 = launch_stats()["umma"]
    y = MF.linear(x, w, b)
    y.backward(g)
    if dt == "bf16":
        assert launch_stats()["umma"] - u0 == 3  # fwd, dX, dW on tcgen05
    _close(y, oracle.linear_fwd(xq, wq, bq), dt, "y")
    _close(x.grad, oracle.linear_dx(gq, wq), dt, "dx")
    _close(w.grad, oracle.linear_dw(xq, gq), dt, "dw")
    _close(b.grad, oracle.linear_db(gq), dt, "db")


F32_TC_CASES = [
    ((512,), 256, 256),        # one wave, K = 8 k-blocks
    ((3, 300), 1000, 520),     # K not a multiple of 32 (TMA zero fill), N tail of a BN=128 tile
    ((2, 640), 768, 3072),     # BERT-like FFN shape, long K
    ((4096,), 1023, 130),      # N, K odd: 16-byte row pitch only in the split planes
]


@pytest.mark.parametrize("case", F32_TC_CASES)
def test_linear_fp32_tensor_cores(case):
    """float32 Linear on tcgen05 kind::tf32 (3xTF32: hi*hi + hi*lo + lo*hi over
    hi / lo planes split once per operand): fwd, dX, dW each one tensor-core
    launch, all within the fp32 bar (rtol 1e-5 vs the f64 oracle)."""
    lead, fin, fout = case
    rng = np.random.default_rng(fin * 7 + fout)
    x, xq = _q(rng.standard_normal(lead + (fin,)), "f32")
    w, wq = _q(rng.standard_normal((fout, fin)) / np.sqrt(fin), "f32")
    b, bq = _q(rng.standard_normal(fout), "f32")
    g, gq = _q(rng.standard_normal(lead + (fout,)), "f32")
    for t in (x, w, b):
        t.requires_grad_(True)
    u0 = launch_stats()["umma"]
    y = MF.linear(x, w, b)
    y.backward(g)
    assert launch_stats()["umma"] - u0 == 3
    _close(y, oracle.linear_fwd(xq, wq, bq), "f32", "y")
    _close(x.grad, oracle.linear_dx(gq, wq), "f32", "dx")
    _close(w.grad, oracle.linear_dw(xq, gq), "f32", "dw")
    _close(b.grad, oracle.linear_db(gq), "f32", "db")


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("shape", [(64, 768, 2), (5, 1000, 3), (64, 300, 1)])
def test_linear_skinny_head(shape, dt):
    """Classifier heads (N not a multiple of 8, long K): fwd on the warp-per-output
    dot kernel, dX / dW on the tile kernel; against the f64 oracle."""
    m, fin, fout = shape
    rng = np.random.default_rng(m + fin + fout)
    x, xq = _q(rng.standard_normal((m, fin)), dt)
    w, wq = _q(rng.standard_normal((fout, fin)) / np.sqrt(fin), dt)
    b, bq = _q(rng.standard_normal(fout), dt)
    g, gq = _q(rng.standard_normal((m, fout)), dt)
    for t in (x, w, b):
        t.requires_grad_(True)
    s0 = launch_stats()["simt"]
    y = MF.linear(x, w, b)
    y.backward(g)
    assert launch_stats()["simt"] - s0 >= 3
    _close(y, oracle.linear_fwd(xq, wq, bq), dt, "y")
    _close(x.grad, oracle.linear_dx(gq, wq), dt, "dx")
    _close(w.grad, oracle.linear_dw(xq, gq), dt, "dw")
    _close(b.grad, oracle.linear_db(gq), dt, "db")


@pytest.mark.parametrize("dt", ["bf16", "fp16", "f32"])
def test_gelu_kernels(dt):
    """ms_gelu_fwd / ms_gelu_bwd against the f64 definition (1 ulp of the
    storage type) and against torch's own gelu kernels (same fp32 formula)."""
    rng = np.random.default_rng(5)
    n = 1 << 20 | 13  # ragged tail
    x, xq = _q(rng.standard_normal(n) * 3, dt)
    g, gq = _q(rng.standard_normal(n), dt)
    MF._ops()  # loads the op library
    ops = torch.ops.memsave
    y = ops.gelu_fwd(x)
    dx = ops.gelu_bwd(g, x)
    _close(y, oracle.gelu_fwd(xq), dt, "gelu y")
    _close(dx, oracle.gelu_bwd(gq, xq), dt, "gelu dx")
    ty = torch.nn.functional.gelu(x)
    tdx = torch.ops.aten.gelu_backward(g, x)
    for ours, stock in ((y, ty), (dx, tdx)):
        same = (ours == stock).float().mean().item()
        print(dt, "bit-identical to torch:", same)
        torch.testing.assert_close(ours, stock, rtol=2 ** -7 if dt != "f32" else 1e-6,
                                   atol=1e-6)
    # the forward's erf (interleaved restatement of CUDA's erff) is bit-identical
    # to torch's gelu over every 16-bit input and 16M random fp32 inputs
    if dt == "f32":
        xs = torch.cat([torch.arange(1 << 16, dtype=torch.int32).to(torch.int16)
                        .view(torch.bfloat16).float().to(DEV),
                        torch.randn(1 << 24, device=DEV) * 4])
    else:
        xs = torch.arange(1 << 16, dtype=torch.int32).to(torch.int16).view(TDT[dt]).to(DEV)
    ys, ts = ops.gelu_fwd(xs), torch.nn.functional.gelu(xs)
    both_nan = torch.isnan(ys) & torch.isnan(ts)
    assert bool(((ys == ts) | both_nan).all()), int((~((ys == ts) | both_nan)).sum())


LINEAR_GELU_CASES = [((4096,), 768, 3072), ((3, 100), 200, 72), ((2, 64), 96, 40)]


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("case", LINEAR_GELU_CASES)
def test_linear_gelu(case, dt):
    """Linear -> GELU in one node: the pre-activation equals the Linear's, the
    output is the GELU of the stored pre-activation (GEMM epilogue on the
    tcgen05 path: one launch), and the VJPs match the f64 composition."""
    lead, fin, fout = case
    rng = np.random.default_rng(fin * 3 + fout)
    x, xq = _q(rng.standard_normal(lead + (fin,)), dt)
    w, wq = _q(rng.standard_normal((fout, fin)) / np.sqrt(fin), dt)
    b, bq = _q(rng.standard_normal(fout), dt)
    g, gq = _q(rng.standard_normal(lead + (fout,)), dt)
    MF._ops()
    pre, y0 = torch.ops.memsave.linear_gelu_fwd(x, w, b)
    c0, u0 = launch_count(), launch_stats()["umma"]
    pre2, _ = torch.ops.memsave.linear_gelu_fwd(x, w, b)
    if dt == "bf16" and fin % 8 == 0 and fout % 8 == 0:
        assert launch_count() - c0 == 1 and launch_stats()["umma"] - u0 == 1
    assert torch.equal(pre, pre2)
    assert torch.equal(pre, MF.linear(x, w, b))  # the same GEMM, bit for bit
    _close(pre, oracle.linear_fwd(xq, wq, bq), dt, "pre")
    pq = pre.double().cpu().numpy()
    _close(y0, oracle.gelu_fwd(pq), dt, "y = gelu(pre)")
    assert torch.equal(y0, torch.ops.memsave.gelu_fwd(pre))  # epilogue == elementwise kernel
    for t in (x, w, b):
        t.requires_grad_(True)
    y = MF.linear_gelu(x, w, b)
    assert torch.equal(y.detach(), y0)
    y.backward(g)
    gz = torch.ops.memsave.gelu_bwd(g, pre)
    _close(gz, oracle.gelu_bwd(gq, pq), dt, "dL/dpre")
    zq = gz.double().cpu().numpy()
    _close(x.grad, oracle.linear_dx(zq, wq), dt, "dx")
    _close(w.grad, oracle.linear_dw(xq, zq), dt, "dw")
    _close(b.grad, oracle.linear_db(zq), dt, "db")


LINEAR_DROP_CASES = [((8, 512), 768, 768), ((4, 512), 3072, 768), ((3, 100), 200, 72),
                     ((2, 64), 96, 40)]


@pytest.mark.parametrize("p", [0.1, 0.0])
@pytest.mark.parametrize("case", LINEAR_DROP_CASES)
def test_linear_dropout_add(case, p):
    """Linear -> dropout -> + residual in one node equals the three memsave ops
    bit for bit (forward with the same seed / stream, and every VJP); the
    tcgen05 shapes run it as ONE launch (dropout and add in the epilogue)."""
    lead, fin, fout = case
    rng = np.random.default_rng(fin + 5 * fout)
    x, xq = _q(rng.standard_normal(lead + (fin,)), "bf16")
    w, wq = _q(rng.standard_normal((fout, fin)) / np.sqrt(fin), "bf16")
    b, _ = _q(rng.standard_normal(fout), "bf16")
    r, _ = _q(rng.standard_normal(lead + (fout,)), "bf16")
    g, _ = _q(rng.standard_normal(lead + (fout,)), "bf16")
    seed, stream = 12345, MF.DROPOUT_STREAM_BASE + 3
    MF._ops()
    c0, u0 = launch_count(), launch_stats()["umma"]
    y = MF.linear_dropout_add(x, w, b, r, p, True, seed=seed, stream=stream)
    if fin % 8 == 0 and fout % 8 == 0 and x.numel() // fin >= 128:
        # one GEMM (+ the K-split last wave's finalize, which applies the same steps)
        assert launch_count() - c0 <= 2 and launch_stats()["umma"] - u0 == 1
    ref = MF.dropout(MF.linear(x, w, b), p, True, seed=seed, stream=stream) + r
    assert torch.equal(y, ref)
    if p > 0:  # the mask really drops about p of the elements
        lin = MF.linear(x, w, b)
        frac = ((y == r) & (lin != 0)).float().mean().item()
        assert abs(frac - p) < 0.05, frac
    ts = [t.detach().clone().requires_grad_(True) for t in (x, w, b, r)]
    us = [t.detach().clone().requires_grad_(True) for t in (x, w, b, r)]
    MF.linear_dropout_add(*ts, p, True, seed=seed, stream=stream).backward(g)
    (MF.dropout(MF.linear(*us[:3]), p, True, seed=seed, stream=stream) + us[3]).backward(g)
    for a, c, what in zip(ts, us, ("dx", "dw", "db", "dr")):
        if what in ("dw", "db"):  # fp32 atomics (split-K, column sums): order-dependent
            torch.testing.assert_close(a.grad, c.grad, rtol=2 ** -7, atol=0, msg=what)
        else:
            assert torch.equal(a.grad, c.grad), what
    # eval: no dropout, the Linear (oracle-checked in test_linear) + the residual
    lin = MF.linear(x, w, b)
    _close(lin, oracle.linear_fwd(xq, wq, b.double().cpu().numpy()), "bf16", "linear")
    assert torch.equal(MF.linear_dropout_add(x, w, b, r, p, False), lin + r)


@pytest.mark.parametrize("dt,gen", [("f32", "philox4x32"), ("bf16", "reference"),
                                    ("fp16", "philox4x32")])
def test_linear_dropout_add_other_paths(dt, gen):
    """float32 (3xTF32 GEMM), the reference generator and fp16 run the three
    launches (or fp16's epilogue) and still equal the composed ops bit for bit."""
    rng = np.random.default_rng(17)
    x, _ = _q(rng.standard_normal((3, 128, 256)), dt)
    w, _ = _q(rng.standard_normal((192, 256)) / 16.0, dt)
    b, _ = _q(rng.standard_normal(192), dt)
    r, _ = _q(rng.standard_normal((3, 128, 192)), dt)
    kw = dict(seed=99, stream=MF.DROPOUT_STREAM_BASE + 1, generator=gen)
    y = MF.linear_dropout_add(x, w, b, r, 0.25, True, **kw)
    ref = MF.dropout(MF.linear(x, w, b), 0.25, True, **kw) + r
    assert torch.equal(y, ref)


def test_linear_golden(linbn_golden):
    g = linbn_golden
    for case in ("lin_small", "lin_3d"):
        x, xq = _q(g[f"{case}/x"], "f32")
        w, wq = _q(g[f"{case}/w"], "f32")
        b, bq = _q(g[f"{case}/b"], "f32")
        gy, gq = _q(g[f"{case}/g"], "f32")
        for t in (x, w, b):
            t.requires_grad_(True)
        y = MF.linear(x, w, b)
        y.backward(gy)
        _close(y, oracle.linear_fwd(xq, wq, bq), "f32", f"{case} y")
        _close(x.grad, oracle.linear_dx(gq, wq), "f32", f"{case} dx")
        _close(w.grad, oracle.linear_dw(xq, gq), "f32", f"{case} dw")
        _close(b.grad, oracle.linear_db(gq), "f32", f"{case} db")


# ------------------------------------------------------------------ batchnorm (eval)
@pytest.mark.parametrize("shape", [(2, 64, 7, 9), (3, 5, 4, 3), (4, 256, 14, 14), (2, 24, 8, 8)])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("channels_last", [False, True])
def test_bn_eval(shape, dt, channels_last):
    rng = np.random.default_rng(sum(shape))
    c = shape[1]
    x, xq = _q(rng.standard_normal(shape), dt)
    w, wq = _q(rng.standard_normal(c), dt)
    b, bq = _q(rng.standard_normal(c), dt)
    m, mq = _q(0.1 * rng.standard_normal(c), dt)
    v, vq = _q(0.5 + 1.5 * rng.random(c), dt)
    g, gq = _q(rng.standard_normal(shape), dt)
    if channels_last:
        x = x.contiguous(memory_format=torch.channels_last)
        g = g.contiguous(memory_format=torch.channels_last)
    for t in (x, w, b):
        t.requires_grad_(True)
    eps = 1e-5
    y = MF.batch_norm_eval(x, m, v, w, b, eps)
    y.backward(g)
    _close(y, oracle.bn_eval_fwd(xq, mq, vq, wq, bq, eps), dt, "y", ulps=2.01)
    _close(x.grad, oracle.bn_eval_dx(gq, vq, wq, eps), dt, "dx", ulps=2.01)
    _close(w.grad, oracle.bn_eval_dw(gq, xq, mq, vq, eps), dt, "dw", ulps=2.01)
    _close(b.grad, oracle.bn_eval_db(gq), dt, "db", ulps=2.01)


def test_bn_golden(linbn_golden):
    g = linbn_golden
    for case in ("bn_small", "bn_odd"):
        ts = {k: _q(g[f"{case}/{k}"], "f32") for k in ("x", "w", "b", "mean", "var", "g")}
        x, w, b = ts["x"][0], ts["w"][0], ts["b"][0]
        for t in (x, w, b):
            t.requires_grad_(True)
        eps = float(g[f"{case}/eps"])
        y = MF.batch_norm_eval(x, ts["mean"][0], ts["var"][0], w, b, eps)
        y.backward(ts["g"][0])
        q = {k: v[1] for k, v in ts.items()}
        _close(y, oracle.bn_eval_fwd(q["x"], q["mean"], q["var"], q["w"], q["b"], eps), "f32", "y")
        _close(x.grad, oracle.bn_eval_dx(q["g"], q["var"], q["w"], eps), "f32", "dx")
        _close(w.grad, oracle.bn_eval_dw(q["g"], q["x"], q["mean"], q["var"], eps), "f32", "dw")
        _close(b.grad, oracle.bn_eval_db(q["g"]), "f32", "db")


# ------------------------------------------------------------------ saved set on CUDA
@pytest.mark.parametrize("x_rg,w_rg", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_saved_set_cuda(rules_golden, x_rg, w_rg):
    x = torch.randn(2, 64, 8, 8, device=DEV, dtype=torch.bfloat16).contiguous(
        memory_format=torch.channels_last).requires_grad_(bool(x_rg))
    w = torch.randn(32, 64, 3, 3, device=DEV, dtype=torch.bfloat16).requires_grad_(bool(w_rg))
    packed = []

    def pack(t):
        packed.append(tuple(t.shape))
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        MF.conv2d(x, w, None, 1, 1)
    roles = sorted({(2, 64, 8, 8): "x", (32, 64, 3, 3): "w"}[s] for s in packed)
    exp = [row for row in rules_golden if row["kind"] == "conv2d" and row["policy"] == "memsave"
           and row["x_rg"] == bool(x_rg) and row["w_rg"] == bool(w_rg) and not row["b_rg"]][0]
    assert roles == sorted(r for r, _ in exp["saves"])



# ------------------------------------------------------------------ relu / maxpool
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("channels_last", [False, True])
@pytest.mark.parametrize("inplace", [False, True])
def test_relu_bitmask(dt, channels_last, inplace):
    rng = np.random.default_rng(5)
    x64 = rng.standard_normal((3, 16, 7, 9))
    x64[0, 0, 0, :4] = 0.0  # ties at zero -> mask 0
    x, xq = _q(x64, dt)
    g, gq = _q(rng.standard_normal(x64.shape), dt)
    if channels_last:
        x = x.contiguous(memory_format=torch.channels_last)
    leaf = x.clone().requires_grad_(True)
    h = leaf * 1.0  # non-leaf so that in-place is allowed
    y = MF.relu(h, inplace)
    y.backward(g)
    yr, mr = oracle.relu_fwd(xq)
    np.testing.assert_array_equal(y.detach().float().cpu().numpy(), yr)
    np.testing.assert_array_equal(leaf.grad.float().cpu().numpy(), oracle.relu_bwd(gq, mr))


def test_relu_odd_numel():
    x = torch.randn(1001, device=DEV, dtype=torch.bfloat16, requires_grad=True)
    y = MF.relu(x)
    y.backward(torch.ones_like(y))
    torch.testing.assert_close(y, torch.relu(x.detach()))
    torch.testing.assert_close(x.grad, (x.detach() > 0).to(torch.bfloat16))


def test_maxpool_golden():
    import os
    gd = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "maxpool_ref.npz")))
    for case in ("mp_2x2s2", "mp_3x3s2", "mp_3x3s1", "mp_ties"):
        kh, kw, sh, sw = (int(v) for v in gd[f"{case}/geom"])
        x = torch.tensor(gd[f"{case}/x"], dtype=torch.float32, device=DEV, requires_grad=True)
        y = MF.max_pool2d(x, (kh, kw), (sh, sw), 0)
        y.backward(torch.tensor(gd[f"{case}/g"], dtype=torch.float32, device=DEV))
        np.testing.assert_allclose(y.detach().cpu().double().numpy(), gd[f"{case}/y"], rtol=1e-6)
        np.testing.assert_allclose(x.grad.cpu().double().numpy(), gd[f"{case}/dx"], rtol=1e-5,
                                   atol=1e-6)


@pytest.mark.parametrize("shape,k,s,p", [((4, 64, 56, 56), 3, 2, 1), ((2, 24, 15, 13), 3, 2, 1),
                                          ((2, 8, 9, 9), 2, 2, 0), ((3, 5, 10, 8), 3, 1, 1),
                                          ((2, 64, 28, 28), 2, 2, 0)])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_maxpool_padded(shape, k, s, p, dt):
    rng = np.random.default_rng(sum(shape))
    x, xq = _q(rng.standard_normal(shape), dt)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    y = MF.max_pool2d(x, k, s, p)
    yr, local, flat = oracle.maxpool2d_fwd(xq, k, k, s, s, p, p)
    g, gq = _q(rng.standard_normal(yr.shape), dt)
    y.backward(g)
    np.testing.assert_array_equal(y.detach().float().cpu().double().numpy(), yr)
    _close(x.grad, oracle.maxpool2d_bwd(gq, flat, shape[2], shape[3]), dt, "maxpool dx",
           ulps=2.01)
    # against torch's own max_pool2d on the same values (ties: first occurrence)
    xt = x.detach().float().cpu().requires_grad_(True)
    torch.nn.functional.max_pool2d(xt, k, s, p).backward(g.float().cpu())
    np.testing.assert_allclose(x.grad.float().cpu().numpy(), xt.grad.numpy(), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("shape,k,s,p", [((4, 64, 56, 56), 3, 2, 1), ((2, 24, 15, 13), 3, 2, 1),
                                          ((3, 16, 10, 8), 3, 1, 1)])   # last: fallback passes
@pytest.mark.parametrize("with_bn", [True, False])
def test_maxpool_relu_bwd_fused(shape, k, s, p, with_bn):
    # the stem's conv -> BN -> ReLU -> MaxPool: the ReLU keep mask and the BN
    # scale applied in the maxpool backward's store
    rng = np.random.default_rng(sum(shape) + with_bn)
    x, xq = _q(np.abs(rng.standard_normal(shape)), "bf16")
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    n, c, h, w = shape
    keep = rng.random((n, h, w, c)) < 0.7  # NHWC storage order
    mask = torch.from_numpy(np.packbits(keep.reshape(-1), bitorder="little")).to(DEV)
    bn = None
    if with_bn:
        bn = torch.nn.BatchNorm2d(c).to(DEV, torch.bfloat16).eval()
        bn.running_var.copy_(torch.linspace(0.5, 2.0, c))
        bn.weight.data.copy_(torch.linspace(0.25, 1.5, c))
    y = MF.max_pool2d(x, k, s, p, in_mask=mask, in_bn=bn)
    yr, local, flat = oracle.maxpool2d_fwd(xq, k, k, s, s, p, p)
    g, gq = _q(rng.standard_normal(yr.shape), "bf16")
    y.backward(g)
    dxp = oracle.maxpool2d_bwd(gq, flat, h, w)
    if s == 1:  # no fused kernel: maxpool backward, then ms_bn_relu_bwd (two roundings)
        dxp = oracle.round_to(dxp, "bf16")
    ref = np.where(keep.transpose(0, 3, 1, 2), dxp, 0.0)
    if with_bn:
        var = bn.running_var.double().cpu().numpy()
        sc = oracle.round_to(bn.weight.detach().double().cpu().numpy() / np.sqrt(var + 1e-5),
                             "f32")
        ref = ref * sc.reshape(1, -1, 1, 1)
    _close(x.grad, ref, "bf16", "maxpool+relu dx", ulps=2.01)


@pytest.mark.parametrize("shape", [(2, 8, 40, 70), (1, 8, 16, 64), (3, 8, 33, 17)])
def test_fig1_fp32_tiled_kernel(shape):
    # the specialised float32 8->8 3x3/1 kernels (fwd, dX via flipped weights, dW):
    # fwd / dX on the tcgen05 kind::tf32 kernel when W % 4 == 0 (16-byte TMA row
    # pitch), else the CUDA-core tiled kernel; dW always on the CUDA cores
    rng = np.random.default_rng(shape[2])
    x, xq = _q(rng.standard_normal(shape), "f32")
    w, wq = _q(rng.standard_normal((8, 8, 3, 3)) / 8, "f32")
    g, gq = _q(rng.standard_normal(shape), "f32")
    x.requires_grad_(True)
    w.requires_grad_(True)
    s0 = launch_stats()
    y = MF.conv2d(x, w, None, 1, 1)
    y.backward(g)
    s1 = launch_stats()
    tc = s1["umma"] - s0["umma"]
    assert tc == (2 if shape[3] % 4 == 0 else 0)
    assert s1["simt"] - s0["simt"] + tc >= 3
    _close(y, oracle.conv2d_fwd(xq, wq, 1, 1), "f32", "y")
    _close(x.grad, oracle.conv2d_dx(gq, wq, 1, 1, shape[2], shape[3]), "f32", "dx")
    _close(w.grad, oracle.conv2d_dw(xq, gq, 1, 1, 3, 3), "f32", "dw")


@pytest.mark.parametrize("shape", [(2, 64, 16, 16), (1, 16, 11, 14)])
def test_maxpool_ties_after_relu(shape):
    # post-ReLU activations: many exact zeros, so window ties are the common case
    # (first occurrence in row-major window order wins, numpy_impl.py:60-69)
    rng = np.random.default_rng(7)
    x64 = np.maximum(np.round(rng.standard_normal(shape) * 2) / 2, 0)
    x, xq = _q(x64, "bf16")
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    y = MF.max_pool2d(x, 3, 2, 1)
    yr, local, flat = oracle.maxpool2d_fwd(xq, 3, 3, 2, 2, 1, 1)
    g, gq = _q(rng.standard_normal(yr.shape), "bf16")
    y.backward(g)
    np.testing.assert_array_equal(y.detach().float().cpu().double().numpy(), yr)
    _close(x.grad, oracle.maxpool2d_bwd(gq, flat, shape[2], shape[3]), "bf16", "maxpool dx",
           ulps=2.01)


# ------------------------------------------------------------------ dropout (RNG replay)
@pytest.mark.parametrize("case", ["d_small", "d_half", "d_big"])
def test_dropout_mask_is_the_reference_generator(dropout_golden, case):
    import ctypes
    from paper_2404_12406_b200 import _lib
    g = dropout_golden
    seed, stream = (int(v) for v in g[f"{case}/key"])
    p = float(g[f"{case}/p"])
    mask = g[f"{case}/mask"].astype(bool)
    n = mask.size
    x = torch.ones(n, device=DEV, dtype=torch.float32)
    y = MF.dropout(x, p, True, seed=seed, stream=stream, generator="reference")
    np.testing.assert_array_equal((y != 0).cpu().numpy(), mask)
    scale = np.float32(1.0 / (1.0 - p))
    np.testing.assert_array_equal(y.cpu().numpy()[mask], np.full(mask.sum(), scale))
    # the StoreMask byte output of the same kernel (C ABI)
    L = _lib.lib()
    yb = torch.empty_like(x)
    mb = torch.empty(n, dtype=torch.uint8, device=DEV)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.ms_dropout_fwd(n, _lib.MS_F32, ctypes.c_void_p(x.data_ptr()),
                            ctypes.c_void_p(yb.data_ptr()), seed, stream, p,
                            _lib.MS_RNG_PHILOX4X64_REF, ctypes.c_void_p(mb.data_ptr()), st) == 0
    np.testing.assert_array_equal(mb.cpu().numpy(), mask.astype(np.uint8))


@pytest.mark.parametrize("gen", ["philox4x32", "reference"])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("n", [(1 << 20) + 3, 4096 + 13])
def test_dropout_replayed_gradient(dt, n, gen):
    rng = np.random.default_rng(n)
    seed, stream, p = 987654321 + (1 << 40), 1_000_000 + 5, 0.1
    x, xq = _q(rng.standard_normal(n), dt)
    g, gq = _q(rng.standard_normal(n), dt)
    x.requires_grad_(True)
    u0 = launch_count()
    y = MF.dropout(x, p, True, seed=seed, stream=stream, generator=gen)
    y.backward(g)
    assert launch_count() - u0 == 2  # forward + replayed backward on the native kernels
    mask = oracle.dropout_mask(seed, stream, p, n, gen)
    s = float(np.float32(1.0 / (1.0 - p)))
    np.testing.assert_array_equal((x.grad != 0).cpu().numpy() | (gq == 0), mask | (gq == 0))
    _close(y, np.where(mask, xq * s, 0.0), dt, "dropout y")
    _close(x.grad, np.where(mask, gq * s, 0.0), dt, "dropout dx")


def test_dropout_module_seeds_and_storage():
    from paper_2404_12406_b200.nn import MemSaveDropout
    m = MemSaveDropout(0.5, node=3).train()
    x = torch.randn(1000, device=DEV, requires_grad=True)
    torch.manual_seed(0)
    y1 = m(x)
    torch.manual_seed(0)
    y2 = m(x)
    assert torch.equal(y1, y2)  # reproducible under torch.manual_seed
    y3 = m(x)
    assert not torch.equal(y1, y3)  # a fresh key per call
    m.eval()
    assert m(x) is x


# ------------------------------------------------------------------ layernorm
@pytest.mark.parametrize("shape,dt", [((64, 768), "bf16"), ((5, 7, 24), "f32"),
                                      ((3, 4100), "bf16"), ((2, 3, 1000), "bf16"),
                                      ((33, 2048), "fp16"), ((4, 13), "f32")])
@pytest.mark.parametrize("flags", [(1, 1, 1), (1, 0, 0), (0, 1, 0), (0, 0, 1)])
def test_layernorm(shape, dt, flags):
    rng = np.random.default_rng(sum(shape))
    d = shape[-1]
    x, xq = _q(rng.standard_normal(shape) * 2 + 0.5, dt)
    w, wq = _q(rng.standard_normal(d), dt)
    b, bq = _q(rng.standard_normal(d), dt)
    g, gq = _q(rng.standard_normal(shape), dt)
    for t, f in zip((x, w, b), flags):
        t.requires_grad_(bool(f))
    y = MF.layer_norm(x, (d,), w, b, 1e-5)
    yr, _m, _r = oracle.layernorm_fwd(xq, wq, bq, 1e-5, d)
    _close(y, yr, dt, "ln y", ulps=2.01)
    y.backward(g)
    dxr, dwr, dbr = oracle.layernorm_bwd(gq, xq, wq, 1e-5, d)
    if flags[0]:
        _close(x.grad, dxr, dt, "ln dx", ulps=4.01)
    if flags[1]:
        _close(w.grad, dwr, dt, "ln dw", ulps=2.01)
    if flags[2]:
        _close(b.grad, dbr, dt, "ln db", ulps=2.01)


def test_layernorm_golden(ln_golden):
    for case in ("ln_small", "ln_3d"):
        gd = ln_golden
        x = torch.tensor(gd[f"{case}/x"], dtype=torch.float32, device=DEV, requires_grad=True)
        w = torch.tensor(gd[f"{case}/w"], dtype=torch.float32, device=DEV, requires_grad=True)
        b = torch.tensor(gd[f"{case}/b"], dtype=torch.float32, device=DEV, requires_grad=True)
        d = w.numel()
        y = MF.layer_norm(x, (d,), w, b, 1e-5)
        y.backward(torch.tensor(gd[f"{case}/g"], dtype=torch.float32, device=DEV))
        for t, key in ((y, "y"), (x.grad, "dx"), (w.grad, "dw"), (b.grad, "db")):
            np.testing.assert_allclose(t.detach().double().cpu().numpy(), gd[f"{case}/{key}"],
                                       rtol=2e-5, atol=2e-5)


# ------------------------------------------------------------------ conv_transpose2d
def test_conv_transpose_golden(convt_golden):
    for case in ("ct_s2", "ct_s1"):
        gd = convt_golden
        s, p = (int(v) for v in gd[f"{case}/geom"])
        for dt in ("f32", "bf16"):
            x, xq = _q(gd[f"{case}/x"], dt)
            w, wq = _q(gd[f"{case}/w"], dt)
            gy, gq = _q(gd[f"{case}/g"], dt)
            if dt == "bf16":
                x = x.contiguous(memory_format=torch.channels_last)
            x.requires_grad_(True)
            w.requires_grad_(True)
            y = MF.conv_transpose2d(x, w, None, s, p)
            y.backward(gy)
            _close(y, oracle.conv_transpose2d_fwd(xq, wq, None, s, p), dt, f"{case} y")
            _close(x.grad, oracle.conv_transpose2d_dx(gq, wq, s, p), dt, f"{case} dx")
            _close(w.grad, oracle.conv_transpose2d_dw(xq, gq, s, p, wq.shape[2], wq.shape[3]), dt,
                   f"{case} dw")


@pytest.mark.parametrize("case", [(2, 64, 7, 7, 128, 3, 2, 1, 1), (2, 128, 8, 8, 64, 4, 2, 1, 0),
                                  (1, 32, 9, 9, 16, 3, 1, 1, 0)])
def test_conv_transpose_tcgen05(case):
    n, cin, h, w_, cout, k, s, p, op = case
    rng = np.random.default_rng(cin + cout)
    x, xq = _q(rng.standard_normal((n, cin, h, w_)), "bf16")
    w, wq = _q(rng.standard_normal((cin, cout, k, k)) / np.sqrt(cin * k * k), "bf16")
    b, bq = _q(rng.standard_normal(cout), "bf16")
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    w.requires_grad_(True)
    b.requires_grad_(True)
    y = MF.conv_transpose2d(x, w, b, s, p, op)
    yr = oracle.conv_transpose2d_fwd(xq, wq, bq, s, p, op)
    assert tuple(y.shape) == yr.shape
    g, gq = _q(rng.standard_normal(yr.shape), "bf16")
    u0 = launch_stats()["umma"]
    y.backward(g)
    assert launch_stats()["umma"] - u0 >= 2  # dX and dW on tcgen05
    _close(y, yr, "bf16", "convT y", ulps=2.01)
    _close(x.grad, oracle.conv_transpose2d_dx(gq, wq, s, p), "bf16", "convT dx")
    _close(w.grad, oracle.conv_transpose2d_dw(xq, gq, s, p, k, k), "bf16", "convT dw")
    _close(b.grad, oracle.conv_transpose2d_db(gq), "bf16", "convT db", ulps=2.01)


# ------------------------------------------------------------------ fused conv -> BN-eval -> ReLU
@pytest.mark.parametrize("case", [(2, 64, 14, 14, 128, 3, 1, 1, True), (2, 3, 32, 32, 64, 7, 2, 3, True),
                                  (2, 64, 11, 20, 64, 3, 1, 1, True), (1, 64, 12, 9, 64, 3, 1, 1, False),
                                  (3, 128, 9, 9, 256, 3, 2, 1, False), (2, 64, 8, 8, 64, 1, 1, 0, True)])
def test_conv_bn_relu_fused(case):
    n, c, h, w, k, r, s, p, with_relu = case
    rng = np.random.default_rng(k + r)
    x, xq = _q(rng.standard_normal((n, c, h, w)), "bf16")
    wt, wq = _q(rng.standard_normal((k, c, r, r)) / np.sqrt(c * r * r), "bf16")
    mean, mq = _q(0.1 * rng.standard_normal(k), "bf16")
    var, vq = _q(0.5 + rng.random(k), "bf16")
    bw, bwq = _q(rng.standard_normal(k), "bf16")
    bb, bbq = _q(rng.standard_normal(k), "bf16")
    conv = torch.nn.Conv2d(c, k, r, s, p, bias=False).to(DEV, torch.bfloat16)
    conv.weight.data.copy_(wt)
    conv.weight.requires_grad_(False)
    bn = torch.nn.BatchNorm2d(k).to(DEV, torch.bfloat16).eval()
    bn.running_mean.copy_(mean)
    bn.running_var.copy_(var)
    bn.weight.data.copy_(bw)
    bn.bias.data.copy_(bb)
    for prm in bn.parameters():
        prm.requires_grad_(False)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    u0 = launch_stats()["umma"]
    y = MF.conv_bn_relu(x, conv, bn, with_relu)
    assert launch_stats()["umma"] - u0 == 1  # one fused launch
    # oracle: conv in f64, BN affine on the unrounded conv output (the fused epilogue
    # applies it in fp32 before the single rounding), then ReLU
    conv_ref = oracle.conv2d_fwd(xq, wq, s, p)
    sc = bwq / np.sqrt(vq + 1e-5)
    z = conv_ref * sc.reshape(1, -1, 1, 1) + (bbq - mq * sc).reshape(1, -1, 1, 1)
    keep = z > 0 if with_relu else np.ones_like(z, dtype=bool)
    zr = np.where(keep, z, 0.0)
    _close(y, zr, "bf16", "conv_bn_relu y", ulps=2.01)
    g, gq = _q(rng.standard_normal(zr.shape), "bf16")
    y.backward(g)
    ym = y.detach().float().cpu().double().numpy()
    if with_relu:
        # dX = conv_dx(g * keep * s): the kernel rounds g*keep*s to bf16 before the dgrad
        keep_gpu = ym > 0
        gc = oracle.round_to(np.where(keep_gpu, gq, 0.0) *
                             oracle.round_to(sc, "f32").reshape(1, -1, 1, 1), "bf16")
        ref = oracle.conv2d_dx(gc, wq, s, p, h, w)
    else:
        # no mask: the BN scale is folded into the weight, dX = conv_dx(g, bf16(W * s))
        wsq = oracle.round_to(wq * oracle.round_to(sc, "f32").reshape(-1, 1, 1, 1), "bf16")
        ref = oracle.conv2d_dx(gq, wsq, s, p, h, w)
    _close(x.grad, ref, "bf16", "conv_bn_relu dx", ulps=2.01)


@pytest.mark.parametrize("case", [(2, 64, 11, 20, 64, 1, True),    # 3x3 halo dgrad
                                  (2, 64, 9, 14, 128, 2, True),    # stride-2 phase GEMM
                                  (2, 128, 7, 7, 128, 1, False),   # folded BN scale
                                  (1, 64, 6, 6, 64, 1, False)])
def test_conv_bn_relu_tee(case):
    # x feeds the conv and a second consumer: the second consumer's gradient is
    # added to dX inside the dgrad epilogue (one rounding of dgrad + addend)
    n, c, h, w, k, s, with_relu = case
    rng = np.random.default_rng(c + k + s)
    x, xq = _q(rng.standard_normal((n, c, h, w)), "bf16")
    wt, wq = _q(rng.standard_normal((k, c, 3, 3)) / np.sqrt(c * 9), "bf16")
    conv = torch.nn.Conv2d(c, k, 3, s, 1, bias=False).to(DEV, torch.bfloat16)
    conv.weight.data.copy_(wt)
    conv.weight.requires_grad_(False)
    bn = torch.nn.BatchNorm2d(k).to(DEV, torch.bfloat16).eval()
    bn.running_mean.copy_(torch.linspace(-0.2, 0.2, k))
    bn.running_var.copy_(torch.linspace(0.5, 2.0, k))
    bn.weight.data.copy_(torch.linspace(0.5, 1.5, k))
    bn.bias.data.copy_(torch.linspace(-0.3, 0.3, k))
    for prm in bn.parameters():
        prm.requires_grad_(False)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    y, xa = MF.conv_bn_relu_tee(x, conv, bn, with_relu)
    assert xa.data_ptr() == x.data_ptr()  # the tee is an alias, not a copy
    vq = oracle.round_to(rng.standard_normal((n, c, h, w)), "bf16")
    v = torch.from_numpy(vq).to(DEV, torch.bfloat16).contiguous(memory_format=torch.channels_last)
    g, gq = _q(rng.standard_normal(tuple(y.shape)), "bf16")
    ((y.float() * g.float()).sum() + (xa.float() * v.float()).sum()).backward()
    vq_ = v.double().cpu().numpy()
    varq = bn.running_var.double().cpu().numpy()
    sc = bn.weight.double().cpu().numpy() / np.sqrt(varq + 1e-5)
    ym = y.detach().float().cpu().double().numpy()
    if with_relu:
        keep = ym > 0
        gc = oracle.round_to(np.where(keep, gq, 0.0) *
                             oracle.round_to(sc, "f32").reshape(1, -1, 1, 1), "bf16")
        ref = oracle.conv2d_dx(gc, wq, s, 1, h, w)
    else:
        wsq = oracle.round_to(wq * oracle.round_to(sc, "f32").reshape(-1, 1, 1, 1), "bf16")
        ref = oracle.conv2d_dx(gq, wsq, s, 1, h, w)
    _close(x.grad, ref + vq_, "bf16", "tee dx", ulps=2.01)


@pytest.mark.parametrize("case", [(2, 64, 11, 20, 64, 1, True, True),     # halo dgrad
                                  (2, 64, 9, 14, 128, 2, True, False),    # phase GEMM s2
                                  (2, 128, 7, 7, 128, 1, False, True),    # generic s1
                                  (1, 64, 6, 6, 64, 1, False, False)])
def test_fused_conv_in_mask(case):
    # x came out of a fused ReLU [after eval-BN bn_in] whose backward (keep bit
    # mask [* s_in]) runs in this conv's dgrad epilogue, after the tee addend
    n, c, h, w, k, s, with_in_bn, tee = case
    rng = np.random.default_rng(c + k + s + 7)
    x, xq = _q(rng.standard_normal((n, c, h, w)), "bf16")
    wt, wq = _q(rng.standard_normal((k, c, 3, 3)) / np.sqrt(c * 9), "bf16")
    conv = torch.nn.Conv2d(c, k, 3, s, 1, bias=False).to(DEV, torch.bfloat16)
    conv.weight.data.copy_(wt)
    conv.weight.requires_grad_(False)

    def frozen_bn(ch, lo):
        bn = torch.nn.BatchNorm2d(ch).to(DEV, torch.bfloat16).eval()
        bn.running_mean.copy_(torch.linspace(-0.2, 0.2, ch))
        bn.running_var.copy_(torch.linspace(0.5, 2.0, ch))
        bn.weight.data.copy_(torch.linspace(lo, 1.5, ch))
        bn.bias.data.copy_(torch.linspace(-0.3, 0.3, ch))
        for prm in bn.parameters():
            prm.requires_grad_(False)
        return bn

    bn = frozen_bn(k, 0.5)
    bn_in = frozen_bn(c, 0.25) if with_in_bn else None
    keep = rng.random((n, h, w, c)) < 0.6  # NHWC storage order of x
    mask = torch.from_numpy(np.packbits(keep.reshape(-1), bitorder="little")).to(DEV)
    keep_nchw = keep.transpose(0, 3, 1, 2)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    y, _, xa = MF.fused_conv(x, conv, bn, False, tee=tee, in_mask=mask, in_bn=bn_in)
    g, gq = _q(rng.standard_normal(tuple(y.shape)), "bf16")
    loss = (y.float() * g.float()).sum()
    vq = np.zeros(xq.shape)
    if tee:
        vq = oracle.round_to(rng.standard_normal(xq.shape), "bf16")
        v = torch.from_numpy(vq).to(DEV, torch.bfloat16)
        loss = loss + (xa.float() * v.float()).sum()
    loss.backward()

    def scale_of(m):
        var = m.running_var.double().cpu().numpy()
        return oracle.round_to(m.weight.double().cpu().numpy() / np.sqrt(var + 1e-5), "f32")

    wsq = oracle.round_to(wq * scale_of(bn).reshape(-1, 1, 1, 1), "bf16")
    ref = oracle.conv2d_dx(gq, wsq, s, 1, h, w) + vq
    ref = np.where(keep_nchw, ref, 0.0)
    if with_in_bn:
        ref = ref * scale_of(bn_in).reshape(1, -1, 1, 1)
    _close(x.grad, ref, "bf16", "in-mask dx", ulps=2.01)


@pytest.mark.parametrize("shape", [(2, 64, 9, 11), (3, 256, 7, 7)])
def test_bn_relu_eval_trainable_affine(shape):
    # BN(eval) with a trainable affine -> ReLU in one pass: y, dX, dW, db against
    # float64 (BN scale rounded to fp32 as in the kernel)
    n, c, h, w = shape
    rng = np.random.default_rng(c + h)
    x, xq = _q(rng.standard_normal(shape), "bf16")
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    bn = torch.nn.BatchNorm2d(c).to(DEV, torch.bfloat16).eval()
    bn.running_mean.copy_(torch.linspace(-0.5, 0.5, c))
    bn.running_var.copy_(torch.linspace(0.5, 2.0, c))
    bn.weight.data.copy_(torch.linspace(0.5, 1.5, c))
    bn.bias.data.copy_(torch.linspace(-0.3, 0.3, c))
    assert MF.bn_relu_fusable(x, bn)
    y = MF.batch_norm_relu_eval(x, bn)
    g, gq = _q(rng.standard_normal(shape), "bf16")
    y.backward(g.contiguous(memory_format=torch.channels_last))
    mu = bn.running_mean.double().cpu().numpy().reshape(1, -1, 1, 1)
    var = bn.running_var.double().cpu().numpy().reshape(1, -1, 1, 1)
    wq = bn.weight.detach().double().cpu().numpy().reshape(1, -1, 1, 1)
    bq = bn.bias.detach().double().cpu().numpy().reshape(1, -1, 1, 1)
    inv = 1.0 / np.sqrt(var + 1e-5)
    z = (xq - mu) * inv * wq + bq
    keep = y.detach().float().cpu().double().numpy() > 0
    _close(y, np.maximum(z, 0), "bf16", "bn_relu y", ulps=2.01)
    gk = np.where(keep, gq, 0.0)
    _close(x.grad, gk * wq * inv, "bf16", "bn_relu dx", ulps=2.01)
    np.testing.assert_allclose(bn.weight.grad.double().cpu().numpy(),
                               (gk * (xq - mu) * inv).sum(axis=(0, 2, 3)), rtol=2e-2, atol=2e-2)
    np.testing.assert_allclose(bn.bias.grad.double().cpu().numpy(), gk.sum(axis=(0, 2, 3)),
                               rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("shape,resid_cl", [((2, 64, 9, 11), True), ((3, 256, 7, 7), False),
                                            ((2, 1024, 5, 3), True)])
def test_bn_add_relu_eval_trainable_affine(shape, resid_cl):
    # a bottleneck tail with a trainable BN affine: relu(bn(x) + r) in one pass; dX, dW,
    # db and the residual's gradient g * keep (bit-exact) from one backward pass
    n, c, h, w = shape
    rng = np.random.default_rng(c + h + 1)
    x, xq = _q(rng.standard_normal(shape), "bf16")
    r, rq = _q(rng.standard_normal(shape), "bf16")
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    r = (r.contiguous(memory_format=torch.channels_last) if resid_cl else r).requires_grad_(True)
    bn = torch.nn.BatchNorm2d(c).to(DEV, torch.bfloat16).eval()
    bn.running_mean.copy_(torch.linspace(-0.5, 0.5, c))
    bn.running_var.copy_(torch.linspace(0.5, 2.0, c))
    bn.weight.data.copy_(torch.linspace(0.5, 1.5, c))
    bn.bias.data.copy_(torch.linspace(-0.3, 0.3, c))
    y = MF.batch_norm_relu_eval(x, bn, r)
    g, gq = _q(rng.standard_normal(shape), "bf16")
    y.backward(g.contiguous(memory_format=torch.channels_last))
    mu = bn.running_mean.double().cpu().numpy().reshape(1, -1, 1, 1)
    var = bn.running_var.double().cpu().numpy().reshape(1, -1, 1, 1)
    wq = bn.weight.detach().double().cpu().numpy().reshape(1, -1, 1, 1)
    bq = bn.bias.detach().double().cpu().numpy().reshape(1, -1, 1, 1)
    inv = 1.0 / np.sqrt(var + 1e-5)
    z = oracle.round_to((xq - mu) * inv * wq + bq, "bf16")
    yd = y.detach().float().cpu().double().numpy()
    # BN output rounded to bf16 before the add (as the unfused chain stores it): allow a
    # couple of bf16 ulps of |z| + |r| for the fp32-vs-f64 scale and the two roundings
    tol = 2.0 ** -6 * (np.abs(z) + np.abs(rq)) + 1e-6
    assert (np.abs(yd - np.maximum(z + rq, 0)) <= tol).all(), "bn_add_relu y"
    keep = yd > 0
    gk = np.where(keep, gq, 0.0)
    np.testing.assert_array_equal(r.grad.float().cpu().double().numpy(), gk)
    _close(x.grad, gk * wq * inv, "bf16", "bn_add_relu dx", ulps=2.01)
    np.testing.assert_allclose(bn.weight.grad.double().cpu().numpy(),
                               (gk * (xq - mu) * inv).sum(axis=(0, 2, 3)), rtol=2e-2, atol=2e-2)
    np.testing.assert_allclose(bn.bias.grad.double().cpu().numpy(), gk.sum(axis=(0, 2, 3)),
                               rtol=2e-2, atol=2e-2)


def test_add_relu():
    rng = np.random.default_rng(3)
    a, aq = _q(rng.standard_normal((2, 32, 9, 9)), "bf16")
    b, bq = _q(rng.standard_normal((2, 32, 9, 9)), "bf16")
    a = a.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    b = b.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    y = MF.add_relu(a, b)
    s = oracle.round_to(aq + bq, "bf16")
    _close(y, np.maximum(s, 0), "bf16", "add_relu y")
    g, gq = _q(rng.standard_normal(s.shape), "bf16")
    y.backward(g)
    ref = np.where(s > 0, gq, 0.0)
    _close(a.grad, ref, "bf16", "add_relu da")
    _close(b.grad, ref, "bf16", "add_relu db")


def test_fused_resnet18_matches_unfused():
    # ResNet-18 with randomised BN statistics: input gradients in bf16 are chaotic
    # (ReLU masks flip near 0), so every bf16 implementation -- stock torch
    # included -- is ~20 % away from the fp32 gradient.  The fused model must be
    # no further from fp32 than stock bf16 is.
    import copy

    import torchvision

    from benchkit.models import randomize_bn_stats
    from paper_2404_12406_b200.nn import convert_to_memory_saving
    torch.manual_seed(0)
    base = torchvision.models.resnet18().eval()
    randomize_bn_stats(base)
    for prm in base.parameters():
        prm.requires_grad_(False)
    cl = torch.channels_last
    models = {
        "fp32": copy.deepcopy(base).to(DEV).to(memory_format=cl),
        "stock": copy.deepcopy(base).to(DEV, torch.bfloat16).to(memory_format=cl),
        "fused": convert_to_memory_saving(copy.deepcopy(base), fuse=True)
        .to(DEV, torch.bfloat16).to(memory_format=cl),
    }
    assert type(models["fused"]).__name__ != "ResNet" or hasattr(models["fused"], "graph")
    x = torch.randn(4, 3, 224, 224, device=DEV).contiguous(memory_format=cl)
    out = {}
    for name, m in models.items():
        xi = x.to(torch.float32 if name == "fp32" else torch.bfloat16).clone().requires_grad_(True)
        y = m(xi)
        y.float().sum().backward()
        out[name] = (y.float(), xi.grad.float())
    ry, rg = out["fp32"]
    err = {k: (((y - ry).norm() / ry.norm()).item(), ((g - rg).norm() / rg.norm()).item())
           for k, (y, g) in out.items() if k != "fp32"}
    assert err["fused"][0] <= 1.2 * err["stock"][0] + 1e-3, err
    assert err["fused"][1] <= 1.2 * err["stock"][1] + 1e-2, err


def test_fused_resnet50_trainable_bn_matches_unfused():
    # the ResNet-101 fine-tuning shape of workload (BN affine trainable everywhere, BN
    # eval, input without grad) on a ResNet-50 at 96x96: every bottleneck tail runs as
    # one BN -> +residual -> ReLU pass.  Output and BN-affine gradients must be no
    # further from fp32 than stock bf16 is.
    import copy

    import torchvision

    from benchkit.models import randomize_bn_stats
    from paper_2404_12406_b200.nn import convert_to_memory_saving
    torch.manual_seed(0)
    base = torchvision.models.resnet50().eval()
    randomize_bn_stats(base)
    for name, prm in base.named_parameters():
        prm.requires_grad_(".bn" in name or "downsample.1" in name or name.startswith("bn1"))
    cl = torch.channels_last
    models = {
        "fp32": copy.deepcopy(base).to(DEV).to(memory_format=cl),
        "stock": copy.deepcopy(base).to(DEV, torch.bfloat16).to(memory_format=cl),
        "fused": convert_to_memory_saving(copy.deepcopy(base), fuse=True)
        .to(DEV, torch.bfloat16).to(memory_format=cl),
    }
    x = torch.randn(4, 3, 96, 96, device=DEV).contiguous(memory_format=cl)
    out = {}
    for name, m in models.items():
        y = m(x.to(torch.float32 if name == "fp32" else torch.bfloat16))
        y.float().sum().backward()
        gw = torch.cat([p.grad.float().flatten() for p in m.parameters() if p.requires_grad])
        out[name] = (y.float(), gw)
    ry, rg = out["fp32"]
    err = {k: (((y - ry).norm() / ry.norm()).item(), ((g - rg).norm() / rg.norm()).item())
           for k, (y, g) in out.items() if k != "fp32"}
    assert err["fused"][0] <= 1.2 * err["stock"][0] + 1e-3, err
    assert err["fused"][1] <= 1.2 * err["stock"][1] + 1e-2, err


@pytest.mark.parametrize("x_rg,r_rg", [(True, True), (True, False), (False, True)])
def test_conv_bn_add_relu_fused(x_rg, r_rg):
    n, c, h, w, k = 2, 64, 10, 10, 64
    rng = np.random.default_rng(17)
    x, xq = _q(rng.standard_normal((n, c, h, w)), "bf16")
    wt, wq = _q(rng.standard_normal((k, c, 3, 3)) / np.sqrt(c * 9), "bf16")
    res, rq = _q(rng.standard_normal((n, k, h, w)), "bf16")
    conv = torch.nn.Conv2d(c, k, 3, 1, 1, bias=False).to(DEV, torch.bfloat16)
    conv.weight.data.copy_(wt)
    conv.weight.requires_grad_(False)
    bn = torch.nn.BatchNorm2d(k).to(DEV, torch.bfloat16).eval()
    bn.running_mean.copy_(torch.linspace(-0.2, 0.2, k))
    bn.running_var.copy_(torch.linspace(0.5, 2.0, k))
    bn.weight.data.copy_(torch.linspace(0.5, 1.5, k))
    bn.bias.data.copy_(torch.linspace(-0.3, 0.3, k))
    for prm in bn.parameters():
        prm.requires_grad_(False)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(x_rg)
    res = res.contiguous(memory_format=torch.channels_last).requires_grad_(r_rg)
    u0 = launch_stats()["umma"]
    y = MF.conv_bn_add_relu(x, conv, bn, res)
    assert launch_stats()["umma"] - u0 == 1
    mq = bn.running_mean.double().cpu().numpy()
    vq = bn.running_var.double().cpu().numpy()
    sc = bn.weight.double().cpu().numpy() / np.sqrt(vq + 1e-5)
    sh = bn.bias.double().cpu().numpy() - mq * sc
    z = oracle.conv2d_fwd(xq, wq, 1, 1) * sc.reshape(1, -1, 1, 1) + sh.reshape(1, -1, 1, 1) + rq
    _close(y, np.maximum(z, 0), "bf16", "conv_bn_add_relu y", ulps=2.01)
    g, gq = _q(rng.standard_normal(z.shape), "bf16")
    y.backward(g)
    keep = y.detach().float().cpu().double().numpy() > 0
    gm = np.where(keep, gq, 0.0)
    if r_rg:
        _close(res.grad, gm, "bf16", "residual grad")
    if x_rg:
        wsq = oracle.round_to(wq * oracle.round_to(sc, "f32").reshape(-1, 1, 1, 1), "bf16")
        _close(x.grad, oracle.conv2d_dx(gm, wsq, 1, 1, h, w), "bf16", "x grad", ulps=2.01)


@pytest.mark.parametrize("rg", [(1, 1, 1), (0, 1, 0), (1, 0, 0)])
def test_conv_relu_fused(rg):
    n, c, h, w, k = 2, 32, 12, 12, 64
    rng = np.random.default_rng(23)
    x, xq = _q(rng.standard_normal((n, c, h, w)), "bf16")
    wt, wq = _q(rng.standard_normal((k, c, 3, 3)) / np.sqrt(c * 9), "bf16")
    b, bq = _q(0.1 * rng.standard_normal(k), "bf16")
    conv = torch.nn.Conv2d(c, k, 3, 1, 1).to(DEV, torch.bfloat16)
    conv.weight.data.copy_(wt)
    conv.bias.data.copy_(b)
    conv.weight.requires_grad_(bool(rg[1]))
    conv.bias.requires_grad_(bool(rg[2]))
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(bool(rg[0]))
    y = MF.conv_relu(x, conv)
    z = oracle.conv2d_fwd(xq, wq, 1, 1) + bq.reshape(1, -1, 1, 1)
    _close(y, np.maximum(z, 0), "bf16", "conv_relu y", ulps=2.01)
    g, gq = _q(rng.standard_normal(z.shape), "bf16")
    y.backward(g)
    keep = y.detach().float().cpu().double().numpy() > 0
    gm = np.where(keep, gq, 0.0)
    if rg[0]:
        _close(x.grad, oracle.conv2d_dx(gm, wq, 1, 1, h, w), "bf16", "conv_relu dx")
    if rg[1]:
        _close(conv.weight.grad, oracle.conv2d_dw(xq, gm, 1, 1, 3, 3), "bf16", "conv_relu dw")
    if rg[2]:
        _close(conv.bias.grad, gm.sum(axis=(0, 2, 3)), "bf16", "conv_relu db", ulps=2.01)
