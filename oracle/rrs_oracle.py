"""CPU oracle for the Rotated Runtime Smooth (RRS) A4W4 linear layer.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module.  The product path
(paper_2409_20361_b200) never imports it and shares no code with it.

It is a plain, slow, obviously-correct NumPy program that follows the paper step by step
in float64 (float32 where DESIGN.md fixes an f32 operation so that integer decisions are
taken in the same precision on both sides).  Citations: P:n = PAPER.md line n (the
paper's LaTeX), S:n = SPEC.md line n; R-numbers are the readings listed in DESIGN.md §3.

Pipeline (P:109 steps 1-3, Eq. 1-4):
  1. rotate:            X~ = X . H_K                 (Eq. 4, unnormalised H, R1/R2/R3)
  2. channel max:       c_j = max_t |X~_tj|          (Eq. 1, over all T tokens, R6)
  3. reorder:           column j' of the reordered X~ is channel perm[j']   (R5)
  4. group max:         s_g = max_{j' in g} c[perm[j']], 0 -> 1        (P:103(2), R8)
  5. smooth:            Z = X~_perm . fl(1/s_g)       (Eq. 2 P:91 "X/s", R9)
  6. per-token RTN:     alpha_t = m_t/7, q = rint_even(Z . fl(7/m_t))  (R9-R12)
  7. weights (offline): W~ = W.H, permuted, per-row RTN (R13)
  8. group partials:    P_g = sum_{j' in g} q . qw   (int, exact; P:99, P:103(3))
  9. scale-accumulate:  Y = (sum_g s_g P_g) . alpha_t . beta_n / K     (P:99, P:103(3), R1)

Parity status: every function here is pinned by tests/test_oracle_*.py (closed forms,
invariants, SPEC worked examples, brute force, special cases).  The paper's accuracy tables
(Tables 1-4) need models and datasets: "parity unpinned" for those (not implemented here).
"""
from __future__ import annotations

import numpy as np

F32 = np.float32

# ----------------------------------------------------------------------------------------
# Step 1: Hadamard rotation (Eq. 4; App. A.1)
# ----------------------------------------------------------------------------------------


def hadamard_sylvester(n: int) -> np.ndarray:
    """H_n[i][j] = (-1)^popcount(i & j), n = 2^m (Sylvester; entries c_ij in {+1,-1})."""
    if n < 1 or n & (n - 1):
        raise ValueError("Sylvester Hadamard needs a power of two")
    i = np.arange(n, dtype=np.int64)
    a = i[:, None] & i[None, :]
    pc = np.zeros_like(a)
    while a.any():
        pc += a & 1
        a >>= 1
    return np.where(pc & 1, -1, 1).astype(np.int8)


def hadamard_paley28() -> np.ndarray:
    """Paley construction II, q = 13 (R2): H28 = S(x)[[1,-1],[-1,-1]] + I14(x)[[1,1],[1,-1]].

    S = [[0, 1^T], [1, Q]], Q[i][j] = chi_13(j - i) (quadratic character mod 13).
    """
    q = 13
    squares = {(i * i) % q for i in range(1, q)}

    def chi(a: int) -> int:
        a %= q
        return 0 if a == 0 else (1 if a in squares else -1)

    Q = np.array([[chi(j - i) for j in range(q)] for i in range(q)], dtype=np.int64)
    S = np.zeros((q + 1, q + 1), dtype=np.int64)
    S[0, 1:] = 1
    S[1:, 0] = 1
    S[1:, 1:] = Q
    A = np.array([[1, -1], [-1, -1]], dtype=np.int64)
    B = np.array([[1, 1], [1, -1]], dtype=np.int64)
    return (np.kron(S, A) + np.kron(np.eye(q + 1, dtype=np.int64), B)).astype(np.int8)


def hadamard_factor(K: int):
    """K = 2^m -> (1, 2^m);  K = 28 * 2^m -> (28, 2^m);  else unsupported (R2)."""
    if K >= 1 and K & (K - 1) == 0:
        return 1, K
    if K % 28 == 0 and (K // 28) & (K // 28 - 1) == 0:
        return 28, K // 28
    raise ValueError(f"unsupported K={K}: need 2^m or 28*2^m")


def hadamard(K: int) -> np.ndarray:
    """The unnormalised Hadamard matrix H_K (R = H_K / sqrt(K), Eq. 4).

    K = 28*2^m uses H28 (x) H_{2^m}: index i = 2^m * a + b (R2).
    """
    a, b = hadamard_factor(K)
    Hb = hadamard_sylvester(b)
    if a == 1:
        return Hb
    return np.kron(hadamard_paley28().astype(np.int64), Hb.astype(np.int64)).astype(np.int8)


def hadamard_columns(K: int, j0: int, j1: int) -> np.ndarray:
    """Columns [j0, j1) of H_K as float64 (lets rotate() stream H in column blocks)."""
    a, b = hadamard_factor(K)
    i = np.arange(K, dtype=np.int64)[:, None]
    j = np.arange(j0, j1, dtype=np.int64)[None, :]
    lo = i & (b - 1), j & (b - 1)
    x = lo[0] & lo[1]
    pc = np.zeros_like(x)
    while x.any():
        pc += x & 1
        x >>= 1
    h = np.where(pc & 1, -1.0, 1.0)
    if a == 28:
        H28 = hadamard_paley28().astype(np.float64)
        h = h * H28[i // b, j // b]
    return h


def rotate(A: np.ndarray, col_block: int = 1024) -> np.ndarray:
    """X~ = f32_rne(A . H_K), row by row (Eq. 4 P:131 "t_rotation = t . R"; R1/R3).

    A holds bf16 values (float64 array).  Each output element is a sum of +-A_tk; under the
    exactness precondition (exponent span per row <= 45 - ceil(log2 K)) every such sum is
    exact in float64 whatever the order, so one rounding to f32 gives the correctly
    rounded value.  H is streamed in column blocks to bound memory (K=14336: 1.6 GB dense).
    """
    A = np.asarray(A, dtype=np.float64)
    T, K = A.shape
    out = np.empty((T, K), dtype=F32)
    for j0 in range(0, K, col_block):
        j1 = min(K, j0 + col_block)
        out[:, j0:j1] = (A @ hadamard_columns(K, j0, j1)).astype(F32)
    return out


def exactness_span_ok(A: np.ndarray) -> np.ndarray:
    """Per-row check of the exactness precondition (R3): e_max - e_min <= 45 - ceil(log2 K)."""
    A = np.asarray(A, dtype=np.float64)
    K = A.shape[-1]
    lim = 45 - int(np.ceil(np.log2(K)))
    ok = np.ones(A.shape[0], dtype=bool)
    for r in range(A.shape[0]):
        nz = np.abs(A[r][A[r] != 0])
        if nz.size:
            e = np.frexp(nz)[1]
            ok[r] = (e.max() - e.min()) <= lim
    return ok


# ----------------------------------------------------------------------------------------
# Steps 2-4: runtime channel max, reorder, group max (Eq. 1; P:103 (1)-(2))
# ----------------------------------------------------------------------------------------


def channel_max(Xr: np.ndarray) -> np.ndarray:
    """c_j = max_t |X~_tj| over ALL tokens of the call (Eq. 1, R6). No fallback here (R8)."""
    Xr = np.asarray(Xr, dtype=F32)
    if Xr.shape[0] == 0:
        return np.zeros(Xr.shape[1], dtype=F32)
    return np.abs(Xr).max(axis=0).astype(F32)


def perm_from_channel_max(c: np.ndarray) -> np.ndarray:
    """Reorder "according to the magnitude": descending c, ties by ascending index (R5, R21).

    perm[j'] = original (rotated) channel placed at position j'.
    """
    c = np.asarray(c, dtype=np.float64)
    return np.argsort(-c, kind="stable").astype(np.int32)


def group_scales(c: np.ndarray, perm: np.ndarray, L: int) -> np.ndarray:
    """s_g = max_{j' in [gL, gL+L)} c[perm[j']]; s_g == 0 -> 1 ("maximum value of an
    activation group is set as the smoothing scale"; zero fallback R8)."""
    c = np.asarray(c, dtype=F32)
    K = c.shape[0]
    if K % L:
        raise ValueError("K % group != 0 (R7)")
    s = c[np.asarray(perm)].reshape(K // L, L).max(axis=1).astype(F32)
    s[s == 0] = F32(1.0)
    return s


# ----------------------------------------------------------------------------------------
# Steps 5-6: smooth and per-token INT4 RTN (Eq. 2; §2.1)
# ----------------------------------------------------------------------------------------


def quantize_rows(Z: np.ndarray, bits: int = 4):
    """Symmetric RTN per row: alpha = max|Z|/(2^{N-1}-1); q = round_half_even(Z/alpha).

    Pinned f32 semantics (R9/R10/R11): alpha = fl(m/7) is what is stored; the codes use
    r = fl(7/m) and q = clamp(rint_even(fl(Z*r)), -8, 7).  All-zero row: alpha = 1, q = 0 (R8).
    """
    Z = np.asarray(Z, dtype=F32)
    qmax = F32(2 ** (bits - 1) - 1)
    m = np.abs(Z).max(axis=-1) if Z.shape[-1] else np.zeros(Z.shape[:-1], F32)
    m = m.astype(F32)
    nz = m > 0
    safe_m = np.where(nz, m, F32(1.0)).astype(F32)
    alpha = np.where(nz, (safe_m / qmax).astype(F32), F32(1.0)).astype(F32)
    r = (qmax / safe_m).astype(F32)
    t = (Z * r[..., None]).astype(F32)
    q = np.clip(np.rint(t), -(2 ** (bits - 1)), 2 ** (bits - 1) - 1).astype(np.int8)
    q[~nz] = 0
    return q, alpha


def smooth(Xr: np.ndarray, perm: np.ndarray, s: np.ndarray, L: int) -> np.ndarray:
    """Z[t][j'] = fl(X~[t][perm[j']] * fl(1/s_{j'/L}))   (Eq. 2 P:91 "X/s", R9)."""
    Xr = np.asarray(Xr, dtype=F32)
    inv_s = (F32(1.0) / np.asarray(s, dtype=F32)).astype(F32)
    return (Xr[:, np.asarray(perm)] * np.repeat(inv_s, L)[None, :]).astype(F32)


def smooth_quant(Xr, perm, s, L):
    """Steps 5-6 for the activation: (codes int8 [T][K] in reordered order, alpha_t f32 [T])."""
    return quantize_rows(smooth(Xr, perm, s, L))


def pack_int4(q: np.ndarray) -> np.ndarray:
    """byte b of a row = (q[2b] & 0xF) | (q[2b+1] & 0xF) << 4, two's-complement nibbles (D4)."""
    q = np.asarray(q, dtype=np.int16)
    lo = (q[..., 0::2] & 0xF).astype(np.uint8)
    hi = (q[..., 1::2] & 0xF).astype(np.uint8)
    return (lo | (hi << 4)).astype(np.uint8)


def unpack_int4(b: np.ndarray) -> np.ndarray:
    b = np.asarray(b, dtype=np.uint8)
    lo = (b & 0xF).astype(np.int16)
    hi = (b >> 4).astype(np.int16)
    lo = np.where(lo >= 8, lo - 16, lo)
    hi = np.where(hi >= 8, hi - 16, hi)
    out = np.empty(b.shape[:-1] + (b.shape[-1] * 2,), dtype=np.int8)
    out[..., 0::2] = lo
    out[..., 1::2] = hi
    return out


# ----------------------------------------------------------------------------------------
# Step 7: offline weight preparation (permute, never scale)
# ----------------------------------------------------------------------------------------


def prepare_weights(W: np.ndarray, perm: np.ndarray, rotate_w: bool = True):
    """W~ = W.H (offline rotation), columns permuted like X (P:109 step 1, "reorder the
    activation and weight"), per-output-channel RTN (R12, R13: RTN replaces GPTQ).

    Returns (qw int8 [N][K], beta f32 [N], Wr f32 [N][K] before the permutation).
    """
    Wr = rotate(W) if rotate_w else np.asarray(W, dtype=F32)
    qw, beta = quantize_rows(Wr[:, np.asarray(perm)])
    return qw, beta, Wr


# ----------------------------------------------------------------------------------------
# Steps 8-9: grouped integer GEMM and scale-accumulate epilogue (P:103 (3); P:109 3.)
# ----------------------------------------------------------------------------------------


def group_partials(q: np.ndarray, qw: np.ndarray, L: int) -> np.ndarray:
    """P[g][t][n] = sum_{j' in g} q[t][j'] * qw[n][j']  (int32, exact).

    float64 matmul of small integers is exact (|P| <= 128*49 << 2^53); cast back to int32.
    """
    q = np.asarray(q, dtype=np.float64)
    qw = np.asarray(qw, dtype=np.float64)
    T, K = q.shape
    N = qw.shape[0]
    G = K // L
    P = np.empty((G, T, N), dtype=np.int32)
    for g in range(G):
        P[g] = np.rint(q[:, g * L:(g + 1) * L] @ qw[:, g * L:(g + 1) * L].T).astype(np.int32)
    return P


def scale_accumulate(P: np.ndarray, s: np.ndarray, alpha: np.ndarray, beta: np.ndarray,
                     out_scale: float) -> np.ndarray:
    """Y[t][n] = (sum_{g ascending} s_g P_g[t][n]) * alpha_t * beta_n * out_scale, all float64.

    "The runtime smoothing scales are applied to the dequantized interim result" (P:103 (3));
    "Y = s_j . sum X^_j W^_j^T" per block; out_scale = 1/K undoes R = H/sqrt(K) twice (R1).
    """
    acc = np.zeros(P.shape[1:], dtype=np.float64)
    for g in range(P.shape[0]):
        acc += np.float64(s[g]) * P[g].astype(np.float64)
    return acc * np.asarray(alpha, np.float64)[:, None] * np.asarray(beta, np.float64)[None, :] * out_scale


def scale_accumulate_rows(q: np.ndarray, qw: np.ndarray, s, alpha, beta, L: int, out_scale: float):
    """Same as group_partials + scale_accumulate, group by group, without materialising P[G][T][N]."""
    q = np.asarray(q, dtype=np.float64)
    qw = np.asarray(qw, dtype=np.float64)
    acc = np.zeros((q.shape[0], qw.shape[0]), dtype=np.float64)
    for g in range(q.shape[1] // L):
        Pg = q[:, g * L:(g + 1) * L] @ qw[:, g * L:(g + 1) * L].T
        acc += np.float64(s[g]) * Pg
    return acc * np.asarray(alpha, np.float64)[:, None] * np.asarray(beta, np.float64)[None, :] * out_scale


def bf16_round(y: np.ndarray) -> np.ndarray:
    """Correctly rounded (half-even) float64 -> bf16 value, returned as float64 (normal range)."""
    y = np.asarray(y, dtype=np.float64)
    m, e = np.frexp(y)  # y = m * 2^e, 0.5 <= |m| < 1
    scale = np.ldexp(1.0, e - 8)  # bf16 keeps 8 significant bits
    out = np.rint(y / scale) * scale
    return np.where(y == 0, 0.0, out)


# ----------------------------------------------------------------------------------------
# The whole layer and its calibration helper
# ----------------------------------------------------------------------------------------


def subchannel_quant(A: np.ndarray, L: int):
    """Sub-channel symmetric INT4 RTN (the second efficiency baseline of P:322): every row is
    quantised group by group, each group of L consecutive columns with its own scale, by the same per-row rule as
    quantize_rows (R9-R12).  Returns (q int8 [R][K], alpha f32 [G][R])."""
    A = np.asarray(A, dtype=F32)
    R, K = A.shape
    if K % L:
        raise ValueError("K % group != 0")
    q = np.zeros((R, K), dtype=np.int8)
    alpha = np.zeros((K // L, R), dtype=F32)
    for g in range(K // L):
        q[:, g * L:(g + 1) * L], alpha[g] = quantize_rows(A[:, g * L:(g + 1) * L])
    return q, alpha


def subchannel_gemm(q: np.ndarray, qw: np.ndarray, alpha: np.ndarray, beta: np.ndarray, L: int,
                    out_scale: float = 1.0) -> np.ndarray:
    """Y[t][n] = out_scale * sum_g alpha[g][t] * beta[g][n] * P_g[t][n], in float64 (P:322's sub-channel A4W4)."""
    P = group_partials(q, qw, L).astype(np.float64)
    a = np.asarray(alpha, dtype=np.float64)
    b = np.asarray(beta, dtype=np.float64)
    return out_scale * np.einsum("gt,gn,gtn->tn", a, b, P)


def swiglu(g: np.ndarray, u: np.ndarray) -> np.ndarray:
    """LLaMA MLP gate (the paper applies RRS to the up/gate and down_proj inputs of this block,
    P:138): h = silu(g) * u = g / (1 + exp(-g)) * u, in float64 (the definition, written out)."""
    g = np.asarray(g, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    with np.errstate(over="ignore"):
        return g / (1.0 + np.exp(-g)) * u


def calibrate_perm(X_cal: np.ndarray, rotate_x: bool = True) -> np.ndarray:
    """Offline reorder from calibration activations (R5): rotate -> channel max -> sort."""
    Xr = rotate(X_cal) if rotate_x else np.asarray(X_cal, dtype=F32)
    return perm_from_channel_max(channel_max(Xr))


def rrs_linear(X: np.ndarray, W: np.ndarray, perm: np.ndarray, L: int = 128,
               rotate_x: bool = True, prepared=None, keep_partials: bool = True) -> dict:
    """Rotated Runtime Smooth A4W4 linear layer, all intermediates returned.

    X, W: float64 arrays holding bf16 values.  rotate_x=False gives plain Runtime Smooth
    (Eq. 1-3 with group L) and out_scale 1.
    """
    X = np.asarray(X, dtype=np.float64)
    T, K = X.shape
    if K % L:
        raise ValueError("K % group != 0 (R7)")
    Xr = rotate(X) if rotate_x else X.astype(F32)
    c = channel_max(Xr)
    s = group_scales(c, perm, L)
    q, alpha = smooth_quant(Xr, perm, s, L)
    if prepared is None:
        qw, beta, _ = prepare_weights(W, perm, rotate_w=rotate_x)
    else:
        qw, beta = prepared
    out_scale = 1.0 / K if rotate_x else 1.0
    res = dict(Xr=Xr, chan_max=c, s_group=s, q=q, alpha=alpha, Xq=pack_int4(q), qw=qw,
               beta=beta, Wq=pack_int4(qw), out_scale=out_scale)
    if keep_partials:
        P = group_partials(q, qw, L)
        res["P"] = P
        res["Y"] = scale_accumulate(P, s, alpha, beta, out_scale)
    else:
        res["Y"] = scale_accumulate_rows(q, qw, s, alpha, beta, L, out_scale)
    return res
