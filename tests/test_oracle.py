"""Pins for the fp64 oracle (oracle/ffn_oracle.c) against things other than itself.

Each pin is chosen so that a plausible mistake in the oracle fails at least one:
mean vs sum, eps placement, RMS of x vs x*g, W1/W3 swap, transposed weights,
sign of the sigmoid, dropped gain, wrong fold rounding.
"Oracle pins".  No GPU needed.
"""
import json
import math
import os
from decimal import Decimal, getcontext

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from ffn_inputs import make_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def silu(t):
    return t / (1.0 + math.exp(-t))


def _examples():
    with open(GOLDEN) as f:
        return json.load(f)["examples"]


def _f64(a):
    return torch.tensor(a, dtype=torch.float64)


@pytest.mark.parametrize("ex", _examples(), ids=lambda e: e["id"])
def test_worked_examples(ex):
    x, g, w1, w3 = (_f64(ex[k]) for k in ("x", "g", "w1", "w3"))
    out = oracle.ffn(x, g, w1, w3, eps=ex["eps"])
    r = oracle.rms_inv(x, eps=ex["eps"])
    # 1) the stored hand-derived decimal values
    np.testing.assert_allclose(out, np.array(ex["out"]), rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(r, np.array(ex["r"]), rtol=1e-14)
    # 2) the closed form, evaluated independently of the oracle
    if "closed_form" in ex:
        cf = [[eval(ex["closed_form"], {"math": math, "silu": silu})]]
    else:
        cf = [[eval(c, {"math": math, "silu": silu}) for c in ex["closed_form_list"]]]
    np.testing.assert_allclose(out, np.array(cf), rtol=1e-14, atol=1e-15)


def test_zero_w3_gives_exact_zero():
    d = make_inputs(5, 64, 24, family="C", seed=1, dtype="bf16")
    out = oracle.ffn(d["x"], d["g"], d["w1"], torch.zeros_like(d["w3"]))
    assert np.all(out == 0.0)
    out = oracle.ffn(d["x"], d["g"], torch.zeros_like(d["w1"]), d["w3"])
    assert np.all(out == 0.0)


def test_constant_row_closed_form():
    # x = c*1 => r = 1/sqrt(c^2+eps) and RMSNorm(x) = g*c/sqrt(c^2+eps)
    K = 16
    for c, eps in [(2.0, 1e-6), (0.5, 0.25), (3.0, 0.0), (1.0, 3.0)]:
        x = torch.full((1, K), c, dtype=torch.float64)
        r = oracle.rms_inv(x, eps)
        assert r[0] == pytest.approx(1.0 / math.sqrt(c * c + eps), rel=1e-15)


def test_rms_invariant():
    # RMS(RMSNorm(x)/g) = sqrt(ms/(ms+eps)); = 1 exactly-ish at eps = 0
    d = make_inputs(33, 96, 8, family="C", seed=2, dtype="bf16")
    x = d["x"].double().numpy()
    for eps in (0.0, 1e-6, 0.5):
        r = oracle.rms_inv(d["x"], eps)
        rms_normed = np.sqrt(np.mean((x * r[:, None]) ** 2, axis=1))
        ms = np.mean(x * x, axis=1)
        np.testing.assert_allclose(rms_normed, np.sqrt(ms / (ms + eps)), rtol=1e-13)
        if eps == 0.0:
            np.testing.assert_allclose(rms_normed, 1.0, rtol=1e-13)


def test_identity_weights_reproduce_silu_of_rmsnorm():
    # K = N, W1 = W3 = I => out = SiLU(xn) * xn with xn = RMSNorm(x)
    K = 48
    d = make_inputs(7, K, K, family="C", seed=3, dtype="bf16")
    eye = torch.eye(K, dtype=torch.float64)
    out = oracle.ffn(d["x"], d["g"], eye, eye, eps=1e-6)
    xn = F.rms_norm(d["x"].double(), (K,), d["g"].double(), eps=1e-6).numpy()
    np.testing.assert_allclose(out, xn * xn / (1 + np.exp(-xn)), rtol=1e-13, atol=1e-300)


def test_one_hot_rows_select_columns():
    # W1 row n is one-hot at k1(n), W3 row n one-hot at k3(n): h1 = xn[k1], h3 = xn[k3]
    K, N = 40, 17
    d = make_inputs(6, K, N, family="C", seed=4, dtype="bf16")
    rng = np.random.default_rng(0)
    k1, k3 = rng.integers(0, K, N), rng.integers(0, K, N)
    w1 = torch.zeros(N, K, dtype=torch.float64)
    w3 = torch.zeros(N, K, dtype=torch.float64)
    w1[np.arange(N), k1] = 1.0
    w3[np.arange(N), k3] = 1.0
    out = oracle.ffn(d["x"], d["g"], w1, w3, eps=1e-6)
    xn = F.rms_norm(d["x"].double(), (K,), d["g"].double(), eps=1e-6).numpy()
    h1, h3 = xn[:, k1], xn[:, k3]
    np.testing.assert_allclose(out, h1 / (1 + np.exp(-h1)) * h3, rtol=1e-13, atol=1e-300)


@pytest.mark.parametrize("family,dtype", [("A", "bf16"), ("C", "bf16"), ("T", "fp32"), ("L", "bf16")])
def test_matches_torch_float64_library_composition(family, dtype):
    """Special case that reduces to library routines: torch's own rms_norm,
    linear and silu in float64 on the CPU (an independent implementation)."""
    M, K, N = 19, 136, 72
    d = make_inputs(M, K, N, family=family, seed=5, dtype=dtype)
    eps = 1e-6
    x, g, w1, w3 = (d[k].double() for k in ("x", "g", "w1", "w3"))
    xn = F.rms_norm(x, (K,), g, eps=eps)
    ref = (F.silu(F.linear(xn, w1)) * F.linear(xn, w3)).numpy()
    out = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], eps=eps)
    np.testing.assert_allclose(out, ref, rtol=1e-11, atol=1e-14)


def test_brute_force_high_precision_tiny():
    """Brute force in 50-digit decimal arithmetic on a tiny input; the fp64
    oracle must agree to ~1e-13 relative."""
    getcontext().prec = 50
    M, K, N = 3, 8, 5
    d = make_inputs(M, K, N, family="C", seed=6, dtype="bf16")
    eps = Decimal("0.000001")
    X = [[Decimal(float(v)) for v in row] for row in d["x"].double().tolist()]
    G = [Decimal(float(v)) for v in d["g"].double().tolist()]
    W1 = [[Decimal(float(v)) for v in row] for row in d["w1"].double().tolist()]
    W3 = [[Decimal(float(v)) for v in row] for row in d["w3"].double().tolist()]
    out = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], eps=1e-6)
    for m in range(M):
        ms = sum(v * v for v in X[m]) / K
        r = 1 / (ms + eps).sqrt()
        xn = [X[m][k] * r * G[k] for k in range(K)]
        for n in range(N):
            h1 = sum(xn[k] * W1[n][k] for k in range(K))
            h3 = sum(xn[k] * W3[n][k] for k in range(K))
            exact = h1 / (1 + (-h1).exp()) * h3
            assert float(out[m, n]) == pytest.approx(float(exact), rel=1e-12, abs=1e-300)


def test_rows_subset_and_permutation():
    d = make_inputs(21, 64, 40, family="C", seed=7, dtype="bf16")
    full = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"])
    rows = [20, 0, 5, 5, 13]
    sub = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], rows=rows)
    assert np.array_equal(sub, full[rows])
    perm = np.random.default_rng(1).permutation(21)
    outp = oracle.ffn(d["x"][perm], d["g"], d["w1"], d["w3"])
    assert np.array_equal(outp, full[perm])


def test_pow2_scaling_of_x_is_exact_at_eps0():
    # x -> 2^k x with eps = 0 leaves RMSNorm(x) and so out bitwise unchanged
    d = make_inputs(9, 64, 24, family="C", seed=8, dtype="fp32")
    a = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], eps=0.0)
    b = oracle.ffn(d["x"] * 8.0, d["g"], d["w1"], d["w3"], eps=0.0)
    assert np.array_equal(a, b)


def test_w3_scaling_scales_output_exactly():
    d = make_inputs(9, 64, 24, family="C", seed=9, dtype="fp32")
    a = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"])
    b = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"] * 4.0)
    assert np.array_equal(b, 4.0 * a)


# ---- storage rounding used by the fold-aware modes -----------------------------

def test_round_bf16_matches_torch_cast_bitwise():
    rng = np.random.default_rng(10)
    vals = np.concatenate([
        rng.standard_normal(20000).astype(np.float32),
        (rng.standard_normal(20000) * 1e-38).astype(np.float32),      # subnormals
        (rng.standard_normal(2000) * 3e38).astype(np.float32),       # near overflow
        # exact ties: bf16 value + half ulp
        (np.float32(1.0) + np.float32(2.0 ** -8) * np.arange(0, 64, dtype=np.float32)),
        np.array([0.0, -0.0, np.inf, -np.inf], dtype=np.float32),
    ])
    ref = torch.from_numpy(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([oracle.round_bf16_bits(float(v)) for v in vals], dtype=np.uint16)
    assert np.array_equal(got, ref)


def test_round_tf32_ties_and_reference():
    # hand-derived ties (10 explicit mantissa bits; ulp(1) = 2^-10)
    assert oracle.round_tf32(1 + 2 ** -11) == 1.0                         # tie -> even (down)
    assert oracle.round_tf32(1 + 3 * 2 ** -11) == 1 + 2 ** -9             # tie -> even (up)
    assert oracle.round_tf32(1 + 2 ** -11 + 2 ** -20) == 1 + 2 ** -10     # above tie
    assert oracle.round_tf32(-(1 + 3 * 2 ** -11)) == -(1 + 2 ** -9)

    def ref(v):  # Python-float RNE to 11 significant bits (round() is half-even)
        if v == 0:
            return v
        m, e = math.frexp(v)
        return math.ldexp(round(m * 2 ** 11) / 2 ** 11, e)
    rng = np.random.default_rng(11)
    for v in rng.standard_normal(5000).astype(np.float32):
        assert oracle.round_tf32(float(v)) == ref(float(v))


def test_fold_mode_equals_plain_on_exact_fold_families():
    for fam in ("A", "B"):
        d = make_inputs(12, 256, 40, family=fam, seed=12, dtype="bf16")
        plain = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], mode="plain")
        fold = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], mode="fold_bf16")
        np.testing.assert_allclose(fold, plain, rtol=1e-12, atol=1e-15)


def test_fold_mode_equals_plain_on_torch_prefolded_weights():
    """fold_bf16 == plain mode on weights pre-folded by torch's own bf16 cast
    (an independent rounding implementation) with g = 1."""
    d = make_inputs(10, 128, 24, family="C", seed=13, dtype="bf16")
    g = d["g"].float()
    w1f = (d["w1"].float() * g).to(torch.bfloat16)
    w3f = (d["w3"].float() * g).to(torch.bfloat16)
    ones = torch.ones_like(d["g"])
    a = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], mode="fold_bf16")
    b = oracle.ffn(d["x"], ones, w1f, w3f, mode="plain")
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-15)
    # and on full-entropy data the fold really does change the result
    plain = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], mode="plain")
    assert not np.allclose(a, plain, rtol=1e-9, atol=0)


def test_fold_tf32_exact_on_family_T():
    d = make_inputs(16, 64, 128, family="T", seed=14, dtype="fp32")
    plain = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], mode="plain")
    fold = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], mode="fold_tf32")
    np.testing.assert_allclose(fold, plain, rtol=1e-12, atol=1e-15)


def _tf32_rne_py(v: float) -> float:
    """Python-float RNE to 11 significant bits (round() is half-even): an
    implementation independent of the oracle's bit-level rne_f32_bits."""
    if v == 0 or not math.isfinite(v):
        return v
    m, e = math.frexp(v)
    return math.ldexp(round(m * 2 ** 11) / 2 ** 11, e)


def test_fold_tf32_mode_on_full_entropy_fp32():
    """fold_tf32 mode (the fp32 handle's method, R4/R5) on family-C fp32
    data, where the fold's rounding really changes the result: equal to the torch
    float64 composition on weights folded by an independent Python rounding,
    RNE_tf32(RNE_fp32(W*g)), and NOT equal to the plain definition."""
    d = make_inputs(12, 96, 40, family="C", seed=18, dtype="fp32")
    eps = 1e-6
    g = d["g"].double()
    fold = np.vectorize(_tf32_rne_py)
    w1t = torch.from_numpy(fold((d["w1"].double() * g).float().double().numpy()))
    w3t = torch.from_numpy(fold((d["w3"].double() * g).float().double().numpy()))
    x = d["x"].double()
    r = 1.0 / torch.sqrt((x * x).mean(dim=1, keepdim=True) + eps)
    h1 = r * (x @ w1t.T)
    h3 = r * (x @ w3t.T)
    ref = (F.silu(h1) * h3).numpy()
    got = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], eps, mode="fold_tf32")
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-14)
    plain = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], eps, mode="plain")
    # the tf32 fold moves outputs by ~2^-11 relative: far above fp64 rounding
    assert np.max(np.abs(got - plain)) > 1e-6
    # and it is not the bf16 fold either (8 vs 11 significant bits)
    bf = oracle.ffn(d["x"].to(torch.bfloat16), d["g"].to(torch.bfloat16), d["w1"].to(torch.bfloat16),
                    d["w3"].to(torch.bfloat16), eps, mode="fold_bf16")
    assert not np.allclose(got, bf, rtol=1e-6, atol=0)


def test_tolerance_helper():
    ref = np.array([1.0, -2.0, 0.0, 10.0])
    gpu = ref + np.array([0.02, -0.04, 0.001, 0.3])
    worst, nbad, maxerr = oracle.tolerance_ratio(gpu, ref)
    assert nbad == 1 and worst > 1.0                      # 0.3 > 0.2+0.001
    worst, nbad, _ = oracle.tolerance_ratio(np.array([np.nan]), np.array([1.0]))
    assert nbad == 1


def test_tiny_config_runs_fast():
    import time
    d = make_inputs(16, 64, 128, family="T", seed=15, dtype="fp32")
    t0 = time.perf_counter()
    oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], eps=1e-6)
    assert time.perf_counter() - t0 < 1.0


def test_fold_bf16_matches_torch_bitwise():
    d = make_inputs(1, 200, 48, family="C", seed=16, dtype="bf16")
    got = oracle.fold(d["w1"], d["g"])
    ref = (d["w1"].float() * d["g"].float()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)


def test_fold_tf32_reference():
    d = make_inputs(1, 64, 16, family="C", seed=17, dtype="fp32")
    got = oracle.fold(d["w1"], d["g"])
    prod = (d["w1"].double() * d["g"].double()).float().double().numpy()
    ref = np.vectorize(lambda v: 0.0 if v == 0 else math.ldexp(round(math.frexp(v)[0] * 2 ** 11) / 2 ** 11,
                                                               math.frexp(v)[1]))(prod)
    assert np.array_equal(got.astype(np.float64), ref)


# ---- f3: GEMM + LeakyReLU (the paper's mmLeakyReLu) ------------------------

def test_gemm_act_matches_numpy_and_closed_forms():
    rng = np.random.default_rng(20)
    x = rng.standard_normal((7, 40))
    w = rng.standard_normal((9, 40))
    ref = x @ w.T
    np.testing.assert_allclose(oracle.gemm_act(x, w), ref, rtol=1e-12, atol=1e-12)
    lr = oracle.gemm_act(x, w, "leaky_relu", 0.01)
    np.testing.assert_allclose(lr, np.where(ref >= 0, ref, 0.01 * ref), rtol=1e-12, atol=1e-12)
    # negative entries are scaled by exactly alpha (a power of two: bitwise)
    pos = oracle.gemm_act(x, w)
    lr2 = oracle.gemm_act(x, w, "leaky_relu", 0.25)
    assert np.array_equal(lr2, np.where(pos >= 0, pos, 0.25 * pos))
    # alpha = 1 is the identity; identity weights return act(x)
    assert np.array_equal(oracle.gemm_act(x, w, "leaky_relu", 1.0), pos)
    eye = np.eye(40)
    np.testing.assert_array_equal(oracle.gemm_act(x, eye, "leaky_relu", 0.5), np.where(x >= 0, x, 0.5 * x))


def test_gemm_act_paper_shape_bf16_storage():
    d = make_inputs(512, 2048, 512, family="C", seed=21, dtype="bf16")
    out = oracle.gemm_act(d["x"][:8], d["w1"], "leaky_relu", 0.01)
    ref = d["x"][:8].double() @ d["w1"].double().T
    ref = torch.where(ref >= 0, ref, 0.01 * ref).numpy()
    np.testing.assert_allclose(out, ref, rtol=1e-11, atol=1e-12)


# ---- f1: the feed-forward block with its down projection -------------------------

def test_ffn_block_identity_w2_reduces_to_ffn():
    K = N = 48
    d = make_inputs(6, K, N, family="C", seed=22, dtype="bf16")
    eye = torch.eye(K, dtype=torch.float64)
    blk = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], eye)
    np.testing.assert_allclose(blk, oracle.ffn(d["x"], d["g"], d["w1"], d["w3"]), rtol=1e-13, atol=1e-15)


def test_ffn_block_matches_torch_composition_and_is_linear_in_w2():
    M, K, N = 11, 64, 96
    d = make_inputs(M, K, N, family="C", seed=23, dtype="bf16")
    w2 = make_inputs(1, N, K, family="C", seed=24, dtype="bf16")["w1"]   # [K, N]
    x, g, w1, w3 = (d[k].double() for k in ("x", "g", "w1", "w3"))
    xn = F.rms_norm(x, (K,), g, eps=1e-6)
    ref = F.linear(F.silu(F.linear(xn, w1)) * F.linear(xn, w3), w2.double()).numpy()
    blk = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], w2)
    np.testing.assert_allclose(blk, ref, rtol=1e-11, atol=1e-13)
    blk2 = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], (w2.float() * 2).to(torch.bfloat16))
    assert np.array_equal(blk2, 2 * blk)
    # rows subset
    sub = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], w2, rows=[3, 10])
    assert np.array_equal(sub, blk[[3, 10]])


def test_ffn_block_round_hidden_uses_bf16_rne():
    M, K, N = 5, 64, 32
    d = make_inputs(M, K, N, family="C", seed=25, dtype="bf16")
    w2 = torch.zeros(K, N, dtype=torch.float64)
    w2[torch.arange(N), torch.arange(N)] = 1.0          # picks hidden[:, :N] into out[:, :N]
    blk = oracle.ffn_block(d["x"], d["g"], d["w1"], d["w3"], w2, round_hidden=True)
    hid = torch.from_numpy(oracle.ffn(d["x"], d["g"], d["w1"], d["w3"]))
    # torch's independent RNE; both round fp64 -> fp32 -> bf16 (the oracle's documented path)
    ref = hid.float().to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(blk[:, :N], ref)


# ---- f3: stand-alone RMSNorm (the paper's rmsnorm kernel) ------------------

def test_rmsnorm_matches_torch_and_closed_forms():
    d = make_inputs(13, 2048, 8, family="L", seed=26, dtype="bf16")
    out = oracle.rmsnorm(d["x"], d["g"], 1e-6)
    ref = F.rms_norm(d["x"].double(), (2048,), d["g"].double(), eps=1e-6).numpy()
    np.testing.assert_allclose(out, ref, rtol=1e-13, atol=1e-300)
    # E2: rms = 1 exactly, so RMSNorm(x) = x * g
    x = torch.tensor([[1.0, -1.0, 1.0, -1.0]], dtype=torch.float64)
    g = torch.tensor([1.0, 2.0, 0.5, 1.0], dtype=torch.float64)
    assert np.array_equal(oracle.rmsnorm(x, g, 0.0), np.array([[1.0, -2.0, 0.5, -1.0]]))
    # constant row c: RMSNorm = g * c / sqrt(c^2 + eps)
    x = torch.full((1, 8), 3.0, dtype=torch.float64)
    np.testing.assert_allclose(oracle.rmsnorm(x, torch.ones(8, dtype=torch.float64), 7.0), 3.0 / 4.0, rtol=1e-15)
