"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no rotation, no max-smoothing, no
quantisation): it only draws LLaMA-like bf16 activations and N(0, 0.02^2) bf16 weights,
following the recipe in DESIGN.md §4 (SURVEY.md §8(d) "Synthetic inputs").

Why these shapes of outliers (paper citations, PAPER.md line numbers):
  * channel-wise outliers, consistent across tokens, in the inputs of QKV/up/gate
    projections (fig:u_static; "outliers persist in fixed channels");
  * spike outliers ~1000x the token median in the down_proj input, while channel outliers
    there are "not overly large" (fig:spike_num);
  * W is not smoothed by the method, so it carries no outliers.

Every array is returned as raw bf16 bit patterns (np.uint16), so the oracle and the GPU
see the very same bits.  After the bf16 rounding each row is conditioned for the
exactness precondition of DESIGN.md reading R3: |x| < 2^-24 * absmax(row) -> +0.
"""
from __future__ import annotations

import dataclasses

import numpy as np

BASE_SEED = 20240930  # fixed base seed s0

__all__ = [
    "BASE_SEED", "Workload", "WORKLOADS", "f64_to_bf16_bits", "bf16_bits_to_f64",
    "bf16_bits_to_f32", "make_activations", "make_weights", "make_layer",
]


def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round to bf16 (via f32, both steps round-half-even) and return the uint16 bits."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float64).astype(np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(b).astype(np.float64)


def _flush_rows(bits: np.ndarray) -> np.ndarray:
    """|x| < 2^-24 * absmax(row) -> +0 (exactness precondition, R3)."""
    x = bf16_bits_to_f64(bits)
    amax = np.abs(x).max(axis=-1, keepdims=True)
    out = bits.copy()
    out[np.abs(x) < amax * 2.0 ** -24] = 0
    return out


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    T: int
    K: int
    N: int
    profile: str
    group: int = 128
    note: str = ""


# BASELINE.json "configs", numbered C1..C5 in order (SURVEY.md §8(d) "Configs as concrete runs").
WORKLOADS = {
    "c1_tiny": Workload("c1_tiny", 8, 256, 256, "tiny", note="configs[0]"),
    "c2_llama2_7b_qo": Workload("c2_llama2_7b_qo", 2048, 4096, 4096, "channel", note="configs[1]"),
    "c3_llama3_8b_up": Workload("c3_llama3_8b_up", 4096, 4096, 14336, "channel", note="configs[2] up/gate"),
    "c3_llama3_8b_down": Workload("c3_llama3_8b_down", 4096, 14336, 4096, "spike", note="configs[2] down_proj"),
    "c4_decode_t64": Workload("c4_decode_t64", 64, 8192, 8192, "mixed", note="configs[3]"),
    "c4_decode_t1": Workload("c4_decode_t1", 1, 8192, 8192, "mixed", note="configs[3]"),
    "c5_llama3_70b_up": Workload("c5_llama3_70b_up", 8192, 8192, 28672, "channel", note="configs[4]"),
    "c5_llama3_70b_up_rank8": Workload("c5_llama3_70b_up_rank8", 8192, 8192, 3584, "channel",
                                       note="configs[4] per-rank shard at P=8 (N/8 = 3584), one GPU"),
}


def _layer_outliers(profile: str, K: int, layer_seed: int):
    """Per-layer (token-independent) structure: channel scales and outlier channels.

    Shared between the calibration draw and the runtime draw of the same layer, so the
    offline channel reorder sees the same outlier channels as the runtime input.
    """
    rng = np.random.default_rng([layer_seed, K, 1])
    sigma = np.exp(0.5 * rng.standard_normal(K))
    if profile in ("channel", "mixed"):
        n_ch = max(1, K // 256)
        mag_lo, mag_hi = 20.0, 60.0
    elif profile == "spike":
        n_ch = max(1, K // 1024)
        mag_lo, mag_hi = 4.0, 10.0
    elif profile == "tiny":
        n_ch = 0
        mag_lo = mag_hi = 0.0
    else:
        raise ValueError(f"unknown profile {profile!r}")
    ch = rng.choice(K, size=n_ch, replace=False) if n_ch else np.zeros(0, np.int64)
    mags = rng.uniform(mag_lo, mag_hi, size=n_ch)
    signs = np.where(rng.random(n_ch) < 0.5, -1.0, 1.0)
    return sigma, ch, mags, signs


def make_activations(profile: str, T: int, K: int, layer_seed: int, token_seed: int) -> np.ndarray:
    """LLaMA-like activations X[T][K] as bf16 bits (SURVEY.md §8(d) profile table)."""
    if T == 0:
        return np.zeros((0, K), np.uint16)
    sigma, ch, mags, signs = _layer_outliers(profile, K, layer_seed)
    rng = np.random.default_rng([token_seed, T, K, 2])
    x = sigma[None, :] * rng.standard_normal((T, K))
    med_sigma = float(np.median(sigma))
    if ch.size:
        z = rng.standard_normal((T, ch.size))
        x[:, ch] = signs[None, :] * mags[None, :] * med_sigma * np.abs(1.0 + 0.25 * z)
    if profile in ("spike", "mixed"):
        n_tok = max(1, T // 512)
        toks = rng.choice(T, size=min(n_tok, T), replace=False)
        for t in toks:
            n_sp = int(rng.integers(1, 4))
            cols = rng.choice(K, size=n_sp, replace=False)
            med = float(np.median(np.abs(x[t])))
            M = np.exp(rng.uniform(np.log(300.0), np.log(3000.0), size=n_sp))
            sgn = np.where(rng.random(n_sp) < 0.5, -1.0, 1.0)
            x[t, cols] = sgn * M * med
    if profile == "tiny":
        # exactly one channel outlier (channel 200, x50) and one spike (token 3, channel 17, x1000)
        c_out = 200 % K
        x[:, c_out] *= 50.0
        t_sp, c_sp = 3 % T, 17 % K
        x[t_sp, c_sp] = 1000.0 * float(np.median(np.abs(x[t_sp])))
    return _flush_rows(f64_to_bf16_bits(x))


def make_weights(N: int, K: int, seed: int) -> np.ndarray:
    """W[N][K] ~ N(0, 0.02^2), bf16 bits, no outliers (the method never smooths W)."""
    rng = np.random.default_rng([seed, N, K, 3])
    return _flush_rows(f64_to_bf16_bits(0.02 * rng.standard_normal((N, K))))


def make_layer(w: Workload, index: int = 0, T: int | None = None, N: int | None = None,
               T_cal: int | None = None):
    """(X, W, X_cal) bf16 bits for a workload.

    Seeds: config i uses s0+i for its layer, s0+1000+i for the calibration tokens
    (SURVEY.md §8(d)).  X_cal shares the layer's outlier channels but not its tokens.
    """
    T = w.T if T is None else T
    N = w.N if N is None else N
    seed = BASE_SEED + index
    X = make_activations(w.profile, T, w.K, layer_seed=seed, token_seed=seed)
    W = make_weights(N, w.K, seed=seed)
    tc = T_cal if T_cal is not None else max(64, min(T, 2048))
    X_cal = make_activations(w.profile, tc, w.K, layer_seed=seed, token_seed=BASE_SEED + 1000 + index)
    return X, W, X_cal
