"""Pins for the oracle's smoothing / quantisation / grouped-GEMM steps.

Kinds of pin: golden vectors (tests/golden, each with its citation), SPEC
worked examples, brute force on tiny inputs, closed forms, algebraic identities from the
paper, special cases that reduce to textbook routines, and method-level
trend checks which are sanity only, not parity.
"""
import json
import os

import numpy as np
import pytest

from oracle import rrs_oracle as o
from rrs_synth import WORKLOADS, bf16_bits_to_f64, make_activations, make_layer, make_weights

F32 = np.float32


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _f32eq(a, b):
    """Equality after rounding the printed 9-significant-digit values to f32."""
    return np.array_equal(np.asarray(a, dtype=F32), np.asarray(b, dtype=np.float64).astype(F32))


# ---------------------------------------------------------------- golden vectors

def test_golden_B1(golden_dir):
    g = _load(golden_dir, "survey_appendix_b.json")
    for key in ("B1_L1", "B1_L2"):
        c = g[key]
        r = o.rrs_linear(np.array(c["X"], float), np.array(c["W"], float), np.array(c["perm"]), L=c["L"])
        assert _f32eq(r["s_group"], c["s_group"])
        assert np.array_equal(r["q"], c["q"])
        assert np.array_equal(r["P"], np.array(c["P"]))
        assert np.allclose(r["Y"], c["Y"], rtol=5e-9, atol=0)  # golden printed to 9 significant digits
        if key == "B1_L1":
            for f in ("Xr", "chan_max", "alpha", "beta"):
                assert _f32eq(r[f], c[f]), f
            assert np.array_equal(r["qw"], c["qw"])


def test_golden_B2_full_pipeline(golden_dir):
    c = _load(golden_dir, "survey_appendix_b.json")["B2"]
    X, W = np.array(c["X"], float), np.array(c["W"], float)
    Xr = o.rotate(X)
    assert _f32eq(Xr, c["Xr"])
    cm = o.channel_max(Xr)
    assert _f32eq(cm, c["chan_max"])
    perm = o.perm_from_channel_max(cm)
    assert np.array_equal(perm, c["perm"])
    r = o.rrs_linear(X, W, perm, L=c["L"])
    assert _f32eq(r["s_group"], c["s_group"])
    Z = o.smooth(r["Xr"], perm, r["s_group"], c["L"])
    assert _f32eq(Z, c["Z"])
    assert np.array_equal(r["q"], c["q"]) and np.array_equal(r["qw"], c["qw"])
    assert _f32eq(r["alpha"], c["alpha"]) and _f32eq(r["beta"], c["beta"])
    assert np.array_equal(r["P"], np.array(c["P"]))
    assert np.allclose(r["Y"], c["Y"], rtol=5e-9, atol=0)  # golden printed to 9 significant digits


def test_golden_B3_eq4_spike(golden_dir):
    c = _load(golden_dir, "survey_appendix_b.json")["B3"]
    X = np.array(c["X"], float)
    Xr = o.rotate(X)
    assert _f32eq(Xr, c["Xr"])
    s = o.group_scales(o.channel_max(Xr), np.array(c["perm"]), c["L"])
    assert _f32eq(s, c["s_group"])
    q, _ = o.smooth_quant(Xr, np.array(c["perm"]), s, c["L"])
    assert np.array_equal(q, c["q"])


def test_golden_B4_half_even_tie(golden_dir):
    """fl(fl(1/14)*7) = 0.5 exactly -> code 0 under round-half-even (R10); half-away would give 1."""
    c = _load(golden_dir, "survey_appendix_b.json")["B4"]
    Xr = o.rotate(np.array(c["X"], float))
    assert _f32eq(Xr, c["Xr"])
    s = o.group_scales(o.channel_max(Xr), np.array(c["perm"]), c["L"])
    q, _ = o.smooth_quant(Xr, np.array(c["perm"]), s, c["L"])
    assert np.array_equal(q, c["q"])


# ---------------------------------------------------------------- SPEC worked examples

def test_spec_quantize_examples(golden_dir):
    for ex in _load(golden_dir, "spec_examples.json")["quantize_per_row"]:
        q, a = o.quantize_rows(np.array(ex["Z"], dtype=F32))
        assert np.array_equal(q, ex["q"]), ex["cite"]
        assert _f32eq(a, ex["alpha"]), ex["cite"]


def test_spec_channel_max_examples(golden_dir):
    for ex in _load(golden_dir, "spec_examples.json")["channel_max"]:
        assert _f32eq(o.channel_max(np.array(ex["X"], dtype=F32)), ex["c"]), ex["cite"]


def test_spec_build_plan_examples(golden_dir):
    for ex in _load(golden_dir, "spec_examples.json")["build_plan"]:
        c = np.array(ex["c"], dtype=F32)
        perm = o.perm_from_channel_max(c)
        assert np.array_equal(perm, ex["perm"]), ex["cite"]
        assert _f32eq(o.group_scales(c, perm, ex["L"]), ex["s_group"]), ex["cite"]


def test_spec_apply_smooth_examples(golden_dir):
    for ex in _load(golden_dir, "spec_examples.json")["apply_smooth"]:
        X = np.array(ex["X"], dtype=F32)
        c = o.channel_max(X)
        perm = o.perm_from_channel_max(c)
        Z = o.smooth(X, perm, o.group_scales(c, perm, ex["L"]), ex["L"])
        assert _f32eq(Z, ex["Z"]), ex["cite"]


# ---------------------------------------------------------------- quantiser properties

def test_pack_nibble_order():
    q = np.array([[1, -1, 7, -8, 0, 3]], dtype=np.int8)
    b = o.pack_int4(q)
    assert b.tolist() == [[0xF1, 0x87, 0x30]]
    assert np.array_equal(o.unpack_int4(b), q)


def test_quant_roundtrip_bound_and_range():
    """|Z - alpha q| <= alpha/2 (+ f32 slack) and codes within [-7, 7]."""
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((64, 64)).astype(F32)
    q, a = o.quantize_rows(Z)
    assert q.min() >= -7 and q.max() <= 7
    err = np.abs(Z.astype(np.float64) - a[:, None].astype(np.float64) * q)
    assert np.all(err <= a[:, None] * (0.5 + 1e-6))
    # each row's absmax element maps to +-7
    assert np.all(np.abs(q).max(axis=1) == 7)


def test_quant_scale_equivariance_powers_of_two():
    rng = np.random.default_rng(4)
    Z = rng.standard_normal((8, 32)).astype(F32)
    q1, a1 = o.quantize_rows(Z)
    q2, a2 = o.quantize_rows(Z * F32(8.0))
    assert np.array_equal(q1, q2) and np.array_equal(a1 * F32(8.0), a2)


def test_smoothed_values_bounded_by_one():
    """s_g >= |x~| for every x~ in group g, so |Z| <= 1 (SURVEY §8c pins)."""
    X, W, Xc = make_layer(WORKLOADS["c1_tiny"], T=32)
    Xr = o.rotate(bf16_bits_to_f64(X))
    c = o.channel_max(Xr)
    perm = o.perm_from_channel_max(c)
    Z = o.smooth(Xr, perm, o.group_scales(c, perm, 128), 128)
    assert np.abs(Z).max() <= 1.0


def test_group1_columns_absmax_one():
    """With L = 1 every nonzero column of the smoothed activation has absmax 1; with the
    reciprocal multiply of reading R9, fl(x * fl(1/x)) is 1 or 1 - 2^-24."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((16, 8)).astype(F32)
    c = o.channel_max(X)
    perm = o.perm_from_channel_max(c)
    Z = o.smooth(X, perm, o.group_scales(c, perm, 1), 1)
    assert np.all(np.isin(np.abs(Z).max(axis=0), [F32(1.0), F32(1.0 - 2.0 ** -24)]))


# ---------------------------------------------------------------- GEMM: brute force and identities

def test_grouped_gemm_equals_triple_loop():
    """Y = sum_k (alpha_t q_tk s_g(k)) (beta_n qw_nk) / K (Eq. 3 P:92 with group scales)."""
    X, W, _ = make_layer(WORKLOADS["c1_tiny"], T=4, N=5)
    X, W = bf16_bits_to_f64(X), bf16_bits_to_f64(W)
    L, K = 128, X.shape[1]
    perm = o.calibrate_perm(X)
    r = o.rrs_linear(X, W, perm, L=L)
    q, qw, s, a, b = r["q"], r["qw"], r["s_group"], r["alpha"], r["beta"]
    Y = np.zeros((4, 5))
    for t in range(4):
        for n in range(5):
            tot = 0.0
            for k in range(K):
                tot += float(a[t]) * int(q[t, k]) * float(s[k // L]) * float(b[n]) * int(qw[n, k])
            Y[t, n] = tot / K
    assert np.allclose(r["Y"], Y, rtol=1e-12, atol=1e-15)
    # P_g themselves, brute force
    for g in range(K // L):
        for t in range(4):
            for n in range(5):
                assert r["P"][g, t, n] == sum(int(q[t, k]) * int(qw[n, k]) for k in range(g * L, g * L + L))


def test_single_group_degenerate_case():
    """L = K: one block, Y = s alpha beta P / K."""
    X, W, _ = make_layer(WORKLOADS["c1_tiny"], T=3, N=4)
    X, W = bf16_bits_to_f64(X), bf16_bits_to_f64(W)
    perm = np.arange(256, dtype=np.int32)
    r = o.rrs_linear(X, W, perm, L=256)
    P = r["q"].astype(np.int64) @ r["qw"].astype(np.int64).T
    Y = float(r["s_group"][0]) * P * r["alpha"][:, None].astype(float) * r["beta"][None, :].astype(float) / 256
    assert np.allclose(r["Y"], Y, rtol=1e-13)


def test_unquantized_identity():
    """X W^T = sum_g s_g (X~_g / s_g)(W~_g)^T / K (P:99 + fig:rotate (a) P:52), no quantisation."""
    X, W, _ = make_layer(WORKLOADS["c1_tiny"], T=8, N=16)
    X, W = bf16_bits_to_f64(X), bf16_bits_to_f64(W)
    K, L = 256, 128
    H = o.hadamard(K).astype(np.float64)
    Xr, Wr = X @ H, W @ H
    c = np.abs(Xr).max(axis=0)
    perm = o.perm_from_channel_max(c)
    s = np.array([c[perm[g * L:(g + 1) * L]].max() for g in range(K // L)])
    Y = sum(s[g] * (Xr[:, perm[g * L:(g + 1) * L]] / s[g]) @ Wr[:, perm[g * L:(g + 1) * L]].T for g in range(K // L)) / K
    assert np.abs(Y - X @ W.T).max() / np.abs(X @ W.T).max() < 1e-12


def test_T1_reduces_to_subchannel_quant():
    """T = 1: c = |x~|, so codes are textbook sub-channel absmax INT4 of the rotated, permuted
    token with group scale s_g/7 (SURVEY §8c special cases), up to last-ulp ties."""
    x = bf16_bits_to_f64(make_activations("channel", 1, 512, 21, 22))
    Xr = o.rotate(x)
    c = o.channel_max(Xr)
    perm = o.perm_from_channel_max(c)
    s = o.group_scales(c, perm, 128)
    q, a = o.smooth_quant(Xr, perm, s, 128)
    xp = Xr[0, perm].astype(np.float64)
    pre = xp / (np.repeat(s.astype(np.float64), 128) / 7.0)
    textbook = np.rint(pre)
    near_tie = np.abs(np.abs(pre - np.floor(pre)) - 0.5) < 1e-5
    assert np.array_equal(q[0][~near_tie], textbook[~near_tie])
    assert abs(float(a[0]) - 1 / 7) < 1e-7


def test_G1_reduces_to_per_token_rtn():
    """One group (L = K): s cancels and codes equal per-token RTN of X~ (QuaRot A4 baseline)."""
    x = bf16_bits_to_f64(make_activations("channel", 6, 256, 31, 32))
    Xr = o.rotate(x)
    perm = o.perm_from_channel_max(o.channel_max(Xr))
    s = o.group_scales(o.channel_max(Xr), perm, 256)
    q, _ = o.smooth_quant(Xr, perm, s, 256)
    xp = Xr[:, perm].astype(np.float64)
    pre = xp / (np.abs(xp).max(axis=1, keepdims=True) / 7.0)
    near_tie = np.abs(np.abs(pre - np.floor(pre)) - 0.5) < 1e-4
    assert np.array_equal(q[~near_tie], np.rint(pre)[~near_tie])


def test_identity_data_zero_error():
    """Small-integer X~, W~ already in range give zero quantisation error."""
    Xr = np.array([[7, -3, 2, 7]], dtype=F32)
    Wr = np.array([[1, 2, -7, 7], [7, 0, 0, -7]], dtype=F32)
    perm = np.arange(4, dtype=np.int32)
    s = o.group_scales(o.channel_max(Xr), perm, 4)
    q, a = o.smooth_quant(Xr, perm, s, 4)
    qw, b = o.quantize_rows(Wr)
    Y = o.scale_accumulate(o.group_partials(q, qw, 4), s, a, b, 1.0)
    assert np.allclose(Y, Xr.astype(float) @ Wr.T.astype(float), rtol=1e-6)


def test_zero_inputs_fallbacks():
    """All-zero activation: s_g -> 1, alpha -> 1, codes 0, Y = 0 (R8)."""
    r = o.rrs_linear(np.zeros((3, 256)), bf16_bits_to_f64(make_weights(4, 256, 1)), np.arange(256), L=128)
    assert np.all(r["s_group"] == 1) and np.all(r["alpha"] == 1) and not r["q"].any()
    assert not r["Y"].any()


# ---------------------------------------------------------------- method sanity (trend, not parity)

def _rel_err(r, X, W):
    ref = X @ W.T
    return np.linalg.norm(r["Y"] - ref) / np.linalg.norm(ref)


def test_trend_channel_profile_rrs_beats_rotate_and_rtn():
    """RRS smooths channel-wise outliers better than pure rotation; both beat RTN."""
    X, W, Xc = make_layer(WORKLOADS["c2_llama2_7b_qo"], T=128, N=64, T_cal=128)
    X, W, Xc = bf16_bits_to_f64(X), bf16_bits_to_f64(W)[:, :1024], bf16_bits_to_f64(Xc)
    X, Xc = X[:, :1024], Xc[:, :1024]
    perm = o.calibrate_perm(Xc)
    e_rrs = _rel_err(o.rrs_linear(X, W, perm, L=128), X, W)
    e_rot = _rel_err(o.rrs_linear(X, W, perm, L=1024), X, W)      # one group: pure rotation (QuaRot)
    ident = np.arange(1024, dtype=np.int32)
    e_rtn = _rel_err(o.rrs_linear(X, W, ident, L=1024, rotate_x=False), X, W)
    assert e_rrs <= e_rot < e_rtn


def test_trend_spike_profile_rrs_beats_rs():
    """spikes defeat plain Runtime Smooth (victims); rotation rescues it."""
    bits = make_activations("spike", 256, 1024, 41, 42)
    cal = make_activations("spike", 256, 1024, 41, 43)
    X, Xc = bf16_bits_to_f64(bits), bf16_bits_to_f64(cal)
    W = bf16_bits_to_f64(make_weights(64, 1024, 44))
    e_rrs = _rel_err(o.rrs_linear(X, W, o.calibrate_perm(Xc), L=128), X, W)
    e_rs = _rel_err(o.rrs_linear(X, W, o.calibrate_perm(Xc, rotate_x=False), L=128, rotate_x=False), X, W)
    assert e_rrs < e_rs


def test_keep_partials_false_matches():
    X, W, Xc = make_layer(WORKLOADS["c1_tiny"])
    X, W, Xc = bf16_bits_to_f64(X), bf16_bits_to_f64(W), bf16_bits_to_f64(Xc)
    perm = o.calibrate_perm(Xc)
    a = o.rrs_linear(X, W, perm)
    b = o.rrs_linear(X, W, perm, keep_partials=False)
    assert np.allclose(a["Y"], b["Y"], rtol=1e-14, atol=0)


def test_swiglu_pins():
    """oracle.swiglu against what the definition fixes: silu(0) = 0, the odd-part identity
    silu(x) - silu(-x) = x (x sigma(x) + x sigma(-x) = x), the logistic function from scipy, and the limits."""
    from scipy.special import expit
    rng = np.random.default_rng(7)
    g = rng.normal(0, 4, 1000)
    u = rng.normal(0, 1, 1000)
    assert np.all(o.swiglu(np.zeros(5), np.arange(5.0)) == 0)
    np.testing.assert_allclose(o.swiglu(g, 1.0) - o.swiglu(-g, 1.0), g, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(o.swiglu(g, u), g * expit(g) * u, rtol=1e-13, atol=1e-300)
    assert o.swiglu(np.array([800.0]), np.array([2.0]))[0] == 1600.0
    assert o.swiglu(np.array([-800.0]), np.array([2.0]))[0] == 0.0


def test_subchannel_quant_and_gemm_pins():
    """oracle.subchannel_* (SURVEY §8 f4): brute force on a tiny shape (per-element definition of the group
    scale and code, triple-loop GEMM), and L = K reduces to the per-token / per-channel form."""
    rng = np.random.default_rng(3)
    T, N, K, L = 3, 4, 64, 32
    X = rng.normal(0, 1, (T, K)).astype(np.float32)
    W = rng.normal(0, 0.02, (N, K)).astype(np.float32)
    X[1, 5] = 40.0  # one outlier: only its own group's scale may change
    q, a = o.subchannel_quant(X, L)
    qw, b = o.subchannel_quant(W, L)
    for t in range(T):
        for g in range(K // L):
            m = np.float32(np.max(np.abs(X[t, g * L:(g + 1) * L])))
            assert a[g, t] == np.float32(m / np.float32(7))
            r = np.float32(np.float32(7) / m)
            for j in range(g * L, (g + 1) * L):
                assert q[t, j] == np.clip(np.rint(np.float32(X[t, j] * r)), -8, 7)
    assert a[0, 1] > 4 * a[1, 1]  # the outlier group's scale, not the other group's
    Y = o.subchannel_gemm(q, qw, a, b, L, out_scale=0.5)
    for t in range(T):
        for n in range(N):
            ref = sum(float(a[g, t]) * float(b[g, n]) * sum(int(q[t, j]) * int(qw[n, j]) for j in range(g * L, (g + 1) * L))
                      for g in range(K // L))
            assert np.isclose(Y[t, n], 0.5 * ref, rtol=1e-12, atol=0)
    q1, a1 = o.subchannel_quant(X, K)
    qr, ar = o.quantize_rows(X)
    assert np.array_equal(q1, qr) and np.array_equal(a1[0], ar)
