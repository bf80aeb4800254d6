"""NEXT-1 oracle pins: the retrieval head's front-end (RMSNorm, Q/K projection, RoPE) and the
product's YaRN table (host setup), checked against closed forms and invariants — not against
re-typed copies of the oracle's own formulas.  CPU only."""
import math

import numpy as np
import pytest

import oracle
from paper_2512_00722_b200 import rope


def bits(a):
    """fp32 values that are exactly bf16 -> their bf16 bit patterns."""
    a = np.asarray(a, np.float32)
    u = a.view(np.uint32)
    assert np.all((u & 0xFFFF) == 0), "values must be bf16-representable"
    return (u >> 16).astype(np.uint16)


def vals(b):
    return (np.asarray(b, np.uint32) << 16).view(np.float32)


def rand_bf16(shape, rng, scale=1.0):
    x = (rng.standard_normal(shape) * scale).astype(np.float32)
    return ((x.view(np.uint32) + 0x8000) & 0xFFFF0000).view(np.float32)  # round to a bf16 value


def test_rmsnorm_constant_row_is_the_weight():
    """x = c everywhere: x / rms(x) = sign(c) exactly (eps -> 0), so xn = bf16(w * 1) = w."""
    rng = np.random.default_rng(0)
    H = 256
    w = rand_bf16(H, rng)
    for c in (0.5, -3.0, 1.0):
        x = np.full((1, H), c, np.float32)
        out = oracle.rmsnorm_bf16(bits(x), bits(w), 1e-30)
        want = np.sign(c) * w
        assert np.array_equal(vals(out[0]), want.astype(np.float32))


def test_rmsnorm_scale_invariant_and_unit_weight():
    """eps = 0: scaling x by 2 (exact) leaves xn unchanged; w = None equals w = 1."""
    rng = np.random.default_rng(1)
    x = rand_bf16((3, 512), rng)
    a = oracle.rmsnorm_bf16(bits(x), None, 0.0)
    b = oracle.rmsnorm_bf16(bits(2 * x), None, 0.0)
    c = oracle.rmsnorm_bf16(bits(x), bits(np.ones(512, np.float32)), 0.0)
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_rmsnorm_within_two_bf16_roundings_of_the_exact_value():
    """|xn - w x / sqrt(mean x^2 + eps)| <= 2 bf16 half-ulps (two RN roundings) + tiny."""
    rng = np.random.default_rng(2)
    H = 4096
    x = rand_bf16((4, H), rng, 0.7)
    w = rand_bf16(H, rng) * 0.1 + 1
    w = ((w.view(np.uint32) + 0x8000) & 0xFFFF0000).view(np.float32)
    out = vals(oracle.rmsnorm_bf16(bits(x), bits(w), 1e-5)).reshape(4, H)
    exact = w * x / np.sqrt((x.astype(np.float64) ** 2).mean(1, keepdims=True) + 1e-5)
    assert np.all(np.abs(out - exact) <= np.abs(exact) * (2 ** -8 + 2 ** -8) * 1.01 + 1e-30)


def test_projection_one_hot_input_returns_the_weight_column():
    """xn = e_h, pos = 0, mscale = 1: the rotation is the identity and out = W[:, h] exactly."""
    rng = np.random.default_rng(3)
    N, H, D = 4 * 64, 128, 64
    W = rand_bf16((N, H), rng)
    inv = np.ones(D // 2, np.float32)
    for h in (0, 5, H - 1):
        xn = np.zeros((1, H), np.float32)
        xn[0, h] = 1.0
        out, bound = oracle.rethead_qk(bits(W), bits(xn), inv, [0], D)
        assert np.array_equal(out[0], W[:, h].astype(np.float64))
        assert np.array_equal(bound[0], np.abs(W[:, h]).astype(np.float64))


def test_rotation_quarter_turn_and_norm_preservation():
    """a = fl32(pi/2): (u, v) -> (-v, u) up to cos(fl32(pi/2)) ~ -4e-8; any pos: each pair's
    norm scales by mscale exactly (up to fp64 rounding); pos = 0 with mscale m scales by m."""
    rng = np.random.default_rng(4)
    N, H, D = 2 * 128, 64, 128
    W = rand_bf16((N, H), rng)
    xn = rand_bf16((1, H), rng)
    inv1 = np.ones(D // 2, np.float32)
    base, _ = oracle.rethead_qk(bits(W), bits(xn), inv1, [0], D)
    quarter = np.full(D // 2, np.float32(math.pi / 2), np.float32)
    out, _ = oracle.rethead_qk(bits(W), bits(xn), quarter, [1], D)
    u = base[0].reshape(-1, 2, D // 2)
    o = out[0].reshape(-1, 2, D // 2)
    scale = np.abs(u).max()
    assert np.allclose(o[:, 0], -u[:, 1], atol=1e-7 * scale)
    assert np.allclose(o[:, 1], u[:, 0], atol=1e-7 * scale)
    inv = rope.yarn_inv_freq(D, factor=8.0)[0]
    for pos, m in ((12345, 1.0), (999_999, 1.3)):
        out, _ = oracle.rethead_qk(bits(W), bits(xn), inv, [pos], D, mscale=m)
        o = out[0].reshape(-1, 2, D // 2)
        assert np.allclose((o ** 2).sum(1), m * m * (u ** 2).sum(1), rtol=1e-12)
    out, _ = oracle.rethead_qk(bits(W), bits(xn), inv, [0], D, mscale=1.5)
    assert np.allclose(out[0], 1.5 * base[0], rtol=1e-15)


def test_yarn_table_closed_forms():
    """factor 1: plain RoPE theta_i = base^(-2i/D), mscale 1.  factor s: dimensions whose
    wavelength fits more than beta_fast times in the original context keep theta_i, those
    fitting fewer than beta_slow times get theta_i / s, the band between is in between and
    the table stays monotone; mscale = 1 + 0.1 ln s."""
    D, base = 128, 500000.0
    inv, m = rope.yarn_inv_freq(D, base=base, factor=1.0)
    assert m == 1.0
    assert np.array_equal(inv, (base ** (-2.0 * np.arange(64) / D)).astype(np.float32))
    s, L0 = 16.0, 2048
    inv_s, ms = rope.yarn_inv_freq(D, base=base, factor=s, orig_ctx=L0)
    assert math.isclose(ms, 1 + 0.1 * math.log(16.0), rel_tol=1e-15)
    theta = base ** (-2.0 * np.arange(64) / D)
    fits = L0 * theta / (2 * math.pi)
    hi, lo = fits > 32, fits < 1
    assert hi.any() and lo.any()
    assert np.array_equal(inv_s[hi], theta[hi].astype(np.float32))
    assert np.allclose(inv_s[lo], (theta[lo] / s).astype(np.float32), rtol=1e-7)
    mid = ~(hi | lo)
    assert np.all(inv_s[mid] <= theta[mid] * (1 + 1e-7)) and np.all(inv_s[mid] >= theta[mid] / s * (1 - 1e-7))
    assert np.all(np.diff(inv_s) < 0)
