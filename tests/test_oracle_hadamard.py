"""Pins for the oracle's rotation step (Eq. 4; App. A.1; fig:rotate P:52).

None of these re-type the oracle's formula: they check closed forms, exact integer
orthogonality, an independent recursive construction, exact rational arithmetic and the
paper's invariants.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import rrs_oracle as o
from rrs_synth import bf16_bits_to_f64, make_activations, make_weights


def _recursive_sylvester(n):
    """Independent construction H_{2n} = [[H, H], [H, -H]] (textbook Sylvester)."""
    H = np.array([[1]], dtype=np.int64)
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


@pytest.mark.parametrize("n", [1, 2, 4, 8, 64, 512])
def test_sylvester_matches_recursive_construction(n):
    assert np.array_equal(o.hadamard_sylvester(n).astype(np.int64), _recursive_sylvester(n))


@pytest.mark.parametrize("K", [2, 4, 256, 1024, 28, 28 * 8, 28 * 64])
def test_hadamard_orthogonal_exact_integers(K):
    """H H^T = K I exactly ("R R^T = 1" with R = H/sqrt(K), Eq. 4)."""
    H = o.hadamard(K).astype(np.int64)
    assert set(np.unique(H)) <= {-1, 1}
    assert np.array_equal(H @ H.T, K * np.eye(K, dtype=np.int64))


def test_hadamard_4096_orthogonal_exact():
    H = o.hadamard(4096).astype(np.float64)  # exact: integer entries, sums < 2^53
    assert np.array_equal(H @ H.T, 4096.0 * np.eye(4096))


@pytest.mark.parametrize("K", [14336, 8192])
def test_hadamard_large_rows_orthogonal(K):
    """Sampled rows of H_K against the whole matrix: H[r] . H^T = K e_r (exact in f64)."""
    rng = np.random.default_rng(7)
    rows = rng.choice(K, size=48, replace=False)
    H = o.hadamard(K).astype(np.float64)
    G = H[rows] @ H.T
    expect = np.zeros_like(G)
    expect[np.arange(rows.size), rows] = K
    assert np.array_equal(G, expect)


def test_paley28_symmetric_pm1():
    H28 = o.hadamard_paley28().astype(np.int64)
    assert np.array_equal(H28, H28.T)
    assert set(np.unique(H28)) == {-1, 1}
    assert np.array_equal(H28 @ H28.T, 28 * np.eye(28, dtype=np.int64))


@pytest.mark.parametrize("K", [256, 28 * 16])
def test_streamed_columns_equal_dense(K):
    H = o.hadamard(K).astype(np.float64)
    assert np.array_equal(np.hstack([o.hadamard_columns(K, j, min(K, j + 100)) for j in range(0, K, 100)]), H)


def test_unsupported_K_raises():
    with pytest.raises(ValueError):
        o.hadamard(96 * 3)


def test_rotation_invariance_f64():
    """(X H)(W H)^T = K X W^T  -- fig:rotate (a) P:52 'Y = (XR)(R^-1 W^T) = X W^T'."""
    rng = np.random.default_rng(1)
    K = 256
    X = rng.standard_normal((8, K))
    W = rng.standard_normal((12, K))
    H = o.hadamard(K).astype(np.float64)
    lhs = (X @ H) @ (W @ H).T
    rhs = K * (X @ W.T)
    assert np.abs(lhs - rhs).max() / np.abs(rhs).max() < 1e-12


def test_norm_preservation_and_equal_rows():
    """||t H|| = sqrt(K) ||t|| (orthogonality); equal rows stay equal (fig:rotate (c))."""
    bits = make_activations("channel", 4, 512, 11, 12)
    x = bf16_bits_to_f64(bits)
    x[1] = x[0]
    xr = o.rotate(x).astype(np.float64)
    assert np.array_equal(xr[0], xr[1])
    n0 = np.linalg.norm(x, axis=1) * np.sqrt(512)
    n1 = np.linalg.norm(xr, axis=1)
    assert np.all(np.abs(n1 - n0) / n0 < 1e-6)  # f32 output rounding only


@pytest.mark.parametrize("K,i,O", [(8, 3, 1000.0), (256, 17, -37.5), (28 * 8, 100, 3.0)])
def test_eq4_single_spike_closed_form(K, i, O):
    """Eq. 4: t = O e_i  ->  t . H = O H[i, :], every |entry| = |O| exactly."""
    x = np.zeros((1, K))
    x[0, i] = O
    xr = o.rotate(x).astype(np.float64)[0]
    H = o.hadamard(K).astype(np.float64)
    assert np.array_equal(xr, O * H[i])
    assert np.all(np.abs(xr) == abs(O))


def test_rotation_correctly_rounded_exact_rationals():
    """X~ = f32_rne(exact sum): checked with Python Fractions on generator rows (DESIGN R3)."""
    K = 256
    bits = make_activations("spike", 3, K, 5, 6)
    x = bf16_bits_to_f64(bits)
    xr = o.rotate(x)
    H = _recursive_sylvester(K)
    for t in range(3):
        fr = [Fraction(v) for v in x[t]]
        for j in range(0, K, 37):
            exact = sum(fr[k] * int(H[k, j]) for k in range(K))
            assert np.float32(float(exact)) == xr[t, j]  # exact value fits f64 -> single rounding


def test_generator_meets_exactness_precondition():
    for prof in ("channel", "spike", "mixed", "tiny"):
        x = bf16_bits_to_f64(make_activations(prof, 16, 14336 if prof == "spike" else 4096, 3, 4))
        assert o.exactness_span_ok(x).all()
    w = bf16_bits_to_f64(make_weights(16, 4096, 9))
    assert o.exactness_span_ok(w).all()
