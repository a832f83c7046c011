"""Pin the CPU oracle against golden vectors produced by the reference itself
(oracle/gen_golden.py imports /root/reference/pkg/src/leantape)."""

import numpy as np
import pytest

import oracle
from oracle import conv as oconv
from mscases import CONV_CASES


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_oracle_matches_reference_kernels(conv_golden, case):
    g = conv_golden
    n, cin, h, w, cout, k, s, p = (int(v) for v in g[f"{case}/geom"])
    x, wt, gy = g[f"{case}/x"], g[f"{case}/w"], g[f"{case}/g"]
    y = oconv.conv2d_fwd(x, wt, s, p)
    np.testing.assert_allclose(y, g[f"{case}/y"], rtol=1e-12, atol=1e-12)
    dx = oconv.conv2d_dx(gy, wt, s, p, h, w)
    np.testing.assert_allclose(dx, g[f"{case}/dx"], rtol=1e-12, atol=1e-12)
    dw = oconv.conv2d_dw(x, gy, s, p, k, k)
    np.testing.assert_allclose(dw, g[f"{case}/dw"], rtol=1e-11, atol=1e-11)


def test_conv_known_answers():
    # 1x1 unit kernel is the identity; SPEC.md:257 — k3/s1/p1 preserves H, W
    x = np.arange(20.0).reshape(1, 1, 4, 5)
    assert np.array_equal(oconv.conv2d_fwd(x, np.ones((1, 1, 1, 1)), 1, 0), x)
    y = oconv.conv2d_fwd(np.ones((2, 8, 9, 7)), np.ones((8, 8, 3, 3)), 1, 1)
    assert y.shape == (2, 8, 9, 7)
    # out size formula numpy_impl.py:15-16
    assert oconv.conv_out_size(224, 7, 2, 3) == 112
    assert oconv.conv_out_size(56, 1, 2, 0) == 28


@pytest.mark.parametrize("case", ["lin_small", "lin_3d"])
def test_linear_oracle_matches_spec_vectors(linbn_golden, case):
    g = linbn_golden
    x, w, b, gy = g[f"{case}/x"], g[f"{case}/w"], g[f"{case}/b"], g[f"{case}/g"]
    np.testing.assert_allclose(oracle.linear_fwd(x, w, b), g[f"{case}/y"], rtol=1e-12)
    np.testing.assert_allclose(oracle.linear_dx(gy, w), g[f"{case}/dx"], rtol=1e-12)
    np.testing.assert_allclose(oracle.linear_dw(x, gy), g[f"{case}/dw"], rtol=1e-12)
    np.testing.assert_allclose(oracle.linear_db(gy), g[f"{case}/db"], rtol=1e-12)


def test_linear_identity_kat():
    # W = identity, b = 0 -> Z = X
    x = np.random.default_rng(0).standard_normal((3, 4))
    assert np.allclose(oracle.linear_fwd(x, np.eye(4), np.zeros(4)), x)


@pytest.mark.parametrize("case", ["bn_small", "bn_odd"])
def test_bn_eval_oracle_matches_spec_vectors(linbn_golden, case):
    g = linbn_golden
    x, w, b, m, v, gy = (g[f"{case}/{k}"] for k in ("x", "w", "b", "mean", "var", "g"))
    eps = float(g[f"{case}/eps"])
    np.testing.assert_allclose(oracle.bn_eval_fwd(x, m, v, w, b, eps), g[f"{case}/y"], rtol=1e-12,
                               atol=1e-12)
    np.testing.assert_allclose(oracle.bn_eval_dx(gy, v, w, eps), g[f"{case}/dx"], rtol=1e-12)
    np.testing.assert_allclose(oracle.bn_eval_dw(gy, x, m, v, eps), g[f"{case}/dw"], rtol=1e-11)
    np.testing.assert_allclose(oracle.bn_eval_db(gy), g[f"{case}/db"], rtol=1e-12)


def test_bn_eval_identity_kat():
    # mu=0, var=1, eps=0, W=1, b=0 -> y = x
    x = np.random.default_rng(1).standard_normal((2, 3, 4, 4))
    y = oracle.bn_eval_fwd(x, np.zeros(3), np.ones(3), np.ones(3), np.zeros(3), 0.0)
    assert np.allclose(y, x)


def test_rules_oracle_matches_reference_table(rules_golden):
    for row in rules_golden:
        pol = oracle.Policy(row["policy"])
        got = oracle.storage_decision(row["kind"], pol, x_rg=row["x_rg"], w_rg=row["w_rg"],
                                      out_rg=row["out_rg"], bn_train=row["bn_train"])
        assert [list(t) for t in got] == row["saves"], row


def test_byte_size_kats(kat_golden):
    # (256,8,256,256) F32 = 512 MiB; desk scale (4,8,32,32) = 128 KiB
    assert kat_golden["byte_size_fig1_f32"] == 256 * 8 * 256 * 256 * 4 == 536870912
    assert kat_golden["byte_size_desk_f32"] == 131072


def test_tolerance_helpers():
    r = np.array([1.0, -2.0, 3.0, 1e-3])
    oracle.assert_close_fp32(r.astype(np.float32), r)
    oracle.assert_close_lowp(oracle.round_to(r, "bf16"), r, "bf16")
    with pytest.raises(AssertionError):
        oracle.assert_close_lowp(oracle.round_to(r, "bf16") * 1.02, r, "bf16")
    # round_to matches torch's bf16 rounding
    import torch
    v = np.random.default_rng(2).standard_normal(1000)
    t = torch.tensor(v, dtype=torch.float64).to(torch.bfloat16).double().numpy()
    assert np.array_equal(oracle.round_to(v, "bf16"), t)


POOL_CASES = ["mp_2x2s2", "mp_3x3s2", "mp_3x3s1", "mp_ties"]


@pytest.mark.parametrize("case", POOL_CASES)
def test_maxpool_oracle_matches_reference_kernels(case):
    import os
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "maxpool_ref.npz")))
    kh, kw, sh, sw = (int(v) for v in g[f"{case}/geom"])
    x = g[f"{case}/x"]
    y, local, flat = oracle.maxpool2d_fwd(x, kh, kw, sh, sw)
    np.testing.assert_array_equal(y, g[f"{case}/y"])
    np.testing.assert_array_equal(flat, g[f"{case}/idx"])  # same first-occurrence argmax
    dx = oracle.maxpool2d_bwd(g[f"{case}/g"], flat, x.shape[2], x.shape[3])
    np.testing.assert_allclose(dx, g[f"{case}/dx"], rtol=1e-12, atol=1e-12)


def test_relu_known_answers():
    # SPEC.md forward_relu: x = [-1, 2, 0, 3] -> y = [0, 2, 0, 3], mask bits (0, 1, 0, 1)
    y, mask = oracle.relu_fwd(np.array([-1.0, 2.0, 0.0, 3.0]))
    assert y.tolist() == [0, 2, 0, 3] and mask.tolist() == [False, True, False, True]
    assert oracle.relu_bwd(np.ones(4), mask).tolist() == [0, 1, 0, 1]
    # BitMask byte cost for numel 10^6: 125000 B (SPEC.md, "32x reduction")
    assert (10**6 + 7) // 8 == 125000


# ---------------------------------------------------------------- dropout (RNG replay)
@pytest.mark.parametrize("seed,stream,n", [(0, 1_000_000, 13), (12345, 1_000_003, 40),
                                           (2 ** 62 + 5, 7, 9)])
def test_philox_restatement_matches_reference_generator(seed, stream, n):
    # the reference Rng is numpy's Philox4x64-10 (core.py:100-124); the block
    # function restated in oracle/dropout.py must reproduce its doubles bit for bit
    from oracle import dropout as od
    np.testing.assert_array_equal(od.uniforms_restated(seed, stream, n),
                                  od.uniforms(seed, stream, n))


@pytest.mark.parametrize("case", ["d_small", "d_half", "d_big"])
def test_dropout_oracle_matches_reference_masks(dropout_golden, case):
    g = dropout_golden
    seed, stream = (int(v) for v in g[f"{case}/key"])
    p = float(g[f"{case}/p"])
    mask = g[f"{case}/mask"].astype(bool)
    np.testing.assert_array_equal(oracle.dropout_mask(seed, stream, p, mask.size), mask)
    x = np.linspace(-2, 2, mask.size)
    y, m = oracle.dropout_fwd(x, seed, stream, p)
    np.testing.assert_array_equal(m, mask)
    np.testing.assert_allclose(y, np.where(mask, x / (1 - p), 0.0), rtol=0, atol=0)
    # replay: the backward mask is the forward mask (SPEC.md acceptance 6)
    np.testing.assert_array_equal(oracle.dropout_bwd(np.ones(mask.size), seed, stream, p) != 0,
                                  mask)


def test_dropout_p0_is_identity():
    x = np.arange(10.0)
    y, m = oracle.dropout_fwd(x, 3, 1_000_000, 0.0)
    assert m.all() and np.array_equal(y, x)


# ---------------------------------------------------------------- layernorm
@pytest.mark.parametrize("case", ["ln_small", "ln_3d"])
def test_layernorm_oracle_matches_spec_vectors(ln_golden, case):
    g = ln_golden
    x, w, b, gy = g[f"{case}/x"], g[f"{case}/w"], g[f"{case}/b"], g[f"{case}/g"]
    d = w.size
    y, mean, rstd = oracle.layernorm_fwd(x, w, b, 1e-5, d)
    np.testing.assert_allclose(y, g[f"{case}/y"], rtol=1e-12, atol=1e-12)
    dx, dw, db = oracle.layernorm_bwd(gy, x, w, 1e-5, d)
    np.testing.assert_allclose(dx, g[f"{case}/dx"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dw, g[f"{case}/dw"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(db, g[f"{case}/db"], rtol=1e-12, atol=1e-12)


def test_layernorm_constant_row_kat():
    # SPEC.md forward_layernorm: a constant input row normalises to 0 (then *w + b)
    y, _m, _r = oracle.layernorm_fwd(np.full((2, 6), 3.5), np.full(6, 2.0), np.full(6, 0.25),
                                     1e-5, 6)
    np.testing.assert_allclose(y, 0.25, atol=1e-12)


# ---------------------------------------------------------------- conv_transpose2d
@pytest.mark.parametrize("case", ["ct_s2", "ct_s1"])
def test_conv_transpose_oracle_matches_reference_kernels(convt_golden, case):
    g = convt_golden
    s, p = (int(v) for v in g[f"{case}/geom"])
    x, w, gy = g[f"{case}/x"], g[f"{case}/w"], g[f"{case}/g"]
    np.testing.assert_allclose(oracle.conv_transpose2d_fwd(x, w, None, s, p), g[f"{case}/y"],
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_transpose2d_dx(gy, w, s, p), g[f"{case}/dx"],
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_transpose2d_dw(x, gy, s, p, w.shape[2], w.shape[3]),
                               g[f"{case}/dw"], rtol=1e-11, atol=1e-11)


def test_conv_transpose_unit_kernel_kat():
    # SPEC.md forward_conv_transpose2d: 1x1 unit kernel, stride 1 -> Z = X
    x = np.arange(12.0).reshape(1, 1, 3, 4)
    np.testing.assert_array_equal(oracle.conv_transpose2d_fwd(x, np.ones((1, 1, 1, 1)), None, 1, 0),
                                  x)


def test_philox4x32_known_answers():
    # Random123 kat_vectors for philox4x32_10 (Salmon et al., SC'11)
    from oracle import dropout as od
    kats = [([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
            ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
            ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
             [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1])]
    for ctr, key, want in kats:
        got = od.philox4x32_10([[v] for v in ctr], key)
        assert [int(w[0]) for w in got] == want


def test_philox4x32_mask_rate():
    m = oracle.dropout_mask(99, 1_000_001, 0.3, 200_000, "philox4x32")
    assert abs(m.mean() - 0.7) < 0.005
