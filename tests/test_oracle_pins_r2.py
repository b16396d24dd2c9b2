"""Round-2 pins for oracle functions that round 1 left unpinned (VERDICT r1 "What's weak" 1).

  * bf16_round   -- the bf16 checker behind every bf16 parity assertion.  Pinned against an
                    exact rational rounding written from the format's definition (8 significant bits, ties to
                    even), torch's RNE float32 -> bfloat16 cast, and a hand-written tie table that a
                    half-away-from-zero or a 9-significant-bit rounding fails.
  * exactness_span_ok -- the R3 precondition (per row, exponent span of the nonzero |x| <= 45 - ceil(log2 K)).
                    Pinned at the boundary (limit passes, limit + 1 fails) for K in {128, 4096, 14336}, and
                    against its purpose: at the limit the worst-case row sums exactly in f64 (checked with
                    Fractions), beyond it a crafted row does not.
  * H . H^T = 28672 I on sampled columns (R2: H28 (x) H_1024; the 70B down_proj width).
"""
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import rrs_oracle as o


# ------------------------------------------------------------------------------------------- bf16_round

def _bf16_exact(y: float) -> float:
    """Round-to-nearest-even of y to 8 significant bits, in exact rational arithmetic (normal range)."""
    if y == 0.0:
        return 0.0
    fy = Fraction(y)
    a = abs(fy)
    e = 0  # find e with 2^e <= a < 2^(e+1)
    while a >= 2:
        a /= 2
        e += 1
    while a < 1:
        a *= 2
        e -= 1
    ulp = Fraction(2) ** (e - 7)
    q, r = divmod(abs(fy), ulp)
    if r * 2 > ulp or (r * 2 == ulp and q % 2 == 1):
        q += 1
    v = q * ulp
    return float(-v if fy < 0 else v)


def test_bf16_round_tie_table():
    """Hand-written cases (bf16: 7 fraction bits, ulp(1) = 2^-7)."""
    u = 2.0 ** -7
    cases = [
        (1.0 + u / 2, 1.0),                   # tie, 1 (even) wins; half-away-from-zero gives 1 + u
        (1.0 + 3 * u / 2, 1.0 + 2 * u),       # tie between 1+u (odd) and 1+2u (even)
        (-(1.0 + u / 2), -1.0),               # sign symmetric
        (-(1.0 + 3 * u / 2), -(1.0 + 2 * u)),
        (1.0 + u / 2 + 2.0 ** -40, 1.0 + u),  # just above the tie (double rounding via f32 would give 1)
        (1.0 + u / 2 - 2.0 ** -40, 1.0),      # just below
        (1.0 + u / 4, 1.0),                   # 9 significant bits would keep 1 + u/2 for the next two
        (1.0 + 3 * u / 4, 1.0 + u),
        (255.0, 255.0),                       # 0b11111111: exactly 8 significant bits
        (511.0, 512.0),                       # 9 ones: tie between 510 (odd mantissa) and 512
        (257.0, 256.0),                       # 257: tie between 256 (even) and 258
        (259.0, 260.0),                       # tie between 258 (odd mantissa) and 260
        (3.0 * 2.0 ** -100, 3.0 * 2.0 ** -100),  # exactly representable, tiny
        (1.5 * 2.0 ** 100, 1.5 * 2.0 ** 100),
    ]
    for y, want in cases:
        got = float(o.bf16_round(np.array([y]))[0])
        assert got == want, (y, got, want)
        assert _bf16_exact(y) == want, (y, "tie table itself")


def test_bf16_round_matches_exact_rational_rounding():
    """Random f64 values (not f32-representable: single rounding matters) against the exact definition."""
    rng = np.random.default_rng(11)
    y = rng.standard_normal(4000) * np.exp2(rng.integers(-30, 30, 4000))
    # plus values sitting exactly on, and one f64 ulp either side of, bf16 ties
    base = np.ldexp(rng.integers(128, 256, 2000).astype(np.float64) + 0.5, rng.integers(-20, 20, 2000))
    y = np.concatenate([y, base, np.nextafter(base, np.inf), np.nextafter(base, -np.inf), -base])
    got = o.bf16_round(y)
    want = np.array([_bf16_exact(float(v)) for v in y])
    assert np.array_equal(got, want)


def test_bf16_round_matches_torch_rne_cast_on_f32_values():
    """>= 10^6 f32 values (where one f64 -> bf16 rounding equals torch's f32 -> bf16 RNE), including every
    exact tie pattern (low 16 bits == 0x8000) and random bit patterns over the normal range."""
    rng = np.random.default_rng(12)
    n = 1 << 20
    bits = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    # keep normal, finite f32 (exponent field 1..254) and make a quarter of them exact bf16 ties
    e = (bits >> 23) & 0xFF
    bits = np.where((e == 0) | (e == 255), bits ^ np.uint32(0x40000000), bits).astype(np.uint32)
    bits[: n // 4] = (bits[: n // 4] & np.uint32(0xFFFF0000)) | np.uint32(0x8000)
    x = bits.view(np.float32)
    x = x[np.isfinite(x) & (np.abs(x) >= np.finfo(np.float32).tiny) & (np.abs(x) < 3.3e38)]
    assert x.size > 1_000_000 * 0.99
    want = torch.from_numpy(x.copy()).to(torch.bfloat16).to(torch.float64).numpy()
    got = o.bf16_round(x.astype(np.float64))
    assert np.array_equal(got, want)


# ------------------------------------------------------------------------------------ exactness_span_ok

@pytest.mark.parametrize("K", [128, 4096, 14336])
def test_exactness_span_boundary(K):
    """lim = 45 - ceil(log2 K): a row with span == lim passes, span == lim + 1 fails, zeros are ignored."""
    lim = 45 - int(np.ceil(np.log2(K)))
    assert (K, lim) in ((128, 38), (4096, 33), (14336, 31))
    rows = np.zeros((4, K))
    rows[0, 0], rows[0, 5] = 1.0, 2.0 ** -lim            # frexp exponents 1 and 1 - lim: span lim
    rows[1, 0], rows[1, 5] = 1.0, 2.0 ** -(lim + 1)      # span lim + 1
    rows[2, 0], rows[2, 5] = -1.75, -(2.0 ** -lim) * 1.5  # mantissas do not change the binade
    rows[3, 7] = 3.0                                     # single nonzero: span 0
    assert list(o.exactness_span_ok(rows)) == [True, False, True, True]
    assert o.exactness_span_ok(np.zeros((1, K)))[0]      # all-zero row: vacuous


def test_exactness_span_verdict_example_14336():
    """span 32 at K = 14336 must be rejected (limit 31)."""
    x = np.zeros((1, 14336))
    x[0, 0], x[0, 1] = 2.0 ** 10, 2.0 ** (10 - 32)
    assert not o.exactness_span_ok(x)[0]


def _f64_sum_exact(vals) -> bool:
    acc = 0.0
    for v in vals:
        acc += v
    return Fraction(acc) == sum(Fraction(v) for v in vals)


def test_exactness_limit_is_what_makes_f64_sums_exact():
    """Purpose of the precondition: bf16 inputs (8 significant bits) spanning s binades, K of them, sum exactly
    in f64 whenever 8 + s + ceil(log2 K) <= 53.  At the limit the worst case (every term at the top binade
    with a full mantissa, one at the bottom) is exact in any order; well beyond it a crafted sum is not."""
    K = 128
    lim = 45 - 7
    top = (2.0 - 2.0 ** -7)  # largest bf16 significand, binade 0
    bot = 2.0 ** -lim        # bottom binade
    row = np.zeros((1, K))
    row[0, :-1], row[0, -1] = top, bot
    assert o.exactness_span_ok(row)[0]
    for order in (list(row[0]), list(row[0][::-1])):
        assert _f64_sum_exact(order)
    bad = np.zeros((1, K))
    bad[0, :-1], bad[0, -1] = top, 2.0 ** -(lim + 16)
    assert not o.exactness_span_ok(bad)[0]
    assert not _f64_sum_exact(list(bad[0]))


# -------------------------------------------------------------------------------- H H^T for K = 28672

def test_hadamard_28672_orthogonal_sampled_columns():
    """(H^T H)[:, c] = K e_c for 24 sampled columns c of H_28672 = H28 (x) H_1024 (R2), exact in f64."""
    K = 28672
    rng = np.random.default_rng(28)
    cols = np.sort(rng.choice(K, size=24, replace=False))
    Hs = np.hstack([o.hadamard_columns(K, int(c), int(c) + 1) for c in cols])  # [K][24]
    assert set(np.unique(Hs)) <= {-1.0, 1.0}
    for j0 in range(0, K, 2048):
        Hb = o.hadamard_columns(K, j0, j0 + 2048)
        G = Hb.T @ Hs  # [2048][24] = rows j0.. of H^T H restricted to the sampled columns
        expect = np.zeros_like(G)
        for i, c in enumerate(cols):
            if j0 <= c < j0 + 2048:
                expect[c - j0, i] = K
        assert np.array_equal(G, expect), j0


# -------------------------------------------------------------------------------- Table 4 trend (sanity)

def test_table4_group_size_trend_oracle():
    """Synthetic Table 4: with the paper's group sizes 1, 32, ..., 512 on channel-outlier activations
    (the up/gate input profile), plain Runtime Smooth's error grows with the group size while Rotated Runtime
    Smooth stays flat ("robust to the coarse group scheme").  Method sanity on the oracle, not parity."""
    from rrs_synth import bf16_bits_to_f64, make_activations, make_weights
    K, T, N = 1024, 256, 256
    X = bf16_bits_to_f64(make_activations("channel", T, K, 5, 6))
    W = bf16_bits_to_f64(make_weights(N, K, 7))
    Xc = bf16_bits_to_f64(make_activations("channel", 128, K, 5, 8))
    ref = X @ W.T
    e_rs, e_rrs = [], []
    for L in (1, 32, 64, 128, 256, 512):
        for rot, errs in ((False, e_rs), (True, e_rrs)):
            Y = o.rrs_linear(X, W, o.calibrate_perm(Xc, rotate_x=rot), L=L, rotate_x=rot, keep_partials=False)["Y"]
            errs.append(np.linalg.norm(Y - ref) / np.linalg.norm(ref))
    assert all(b >= a * 0.99 for a, b in zip(e_rs, e_rs[1:])), e_rs
    assert e_rs[-1] > 1.5 * e_rs[1], e_rs
    assert max(e_rrs) < 1.15 * min(e_rrs), e_rrs
    assert e_rrs[-1] < e_rs[-1]
