"""Helpers shared by the GPU parity tests: seeded inputs -> device tensors, oracle references,
and the Y tolerance of DESIGN.md §5 (normalised FP32 error)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import rrs_oracle as o
from rrs_synth import bf16_bits_to_f64

F32 = np.float32


def dev_bf16(bits: np.ndarray, device="cuda") -> torch.Tensor:
    """bf16 bit pattern (uint16 numpy) -> torch.bfloat16 on device, same bits."""
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16))
    return t.to(device).view(torch.bfloat16)


def oracle_layer(X_bits, W_bits, perm, keep_partials=True):
    return o.rrs_linear(bf16_bits_to_f64(X_bits), bf16_bits_to_f64(W_bits), np.asarray(perm), L=128,
                        keep_partials=keep_partials)


def y_normalised_error(Y_gpu: np.ndarray, ref: dict) -> float:
    """max_tn |Y_gpu - Y_or| / (alpha_t beta_n sum_g s_g |P_g[t][n]| / K)   (R15/R18).

    Where the denominator is 0 every P_g is 0 and Y must be exactly 0."""
    P = ref["P"].astype(np.float64)
    s = ref["s_group"].astype(np.float64)
    den = np.tensordot(s, np.abs(P), axes=(0, 0))
    den = den * ref["alpha"].astype(np.float64)[:, None] * ref["beta"].astype(np.float64)[None, :] * ref["out_scale"]
    err = np.abs(Y_gpu.astype(np.float64) - ref["Y"])
    zero = den == 0
    if np.any(err[zero] != 0):
        return np.inf
    return float(np.max(err[~zero] / den[~zero])) if np.any(~zero) else 0.0


def bf16_ulp_error(Y_gpu_bf16: np.ndarray, Y_ref: np.ndarray) -> float:
    """|Y_gpu - bf16(Y_or)| in units of bf16 ulp of Y_or."""
    ref_b = o.bf16_round(Y_ref)
    m, e = np.frexp(np.where(ref_b == 0, 1.0, ref_b))
    ulp = np.ldexp(1.0, e - 8)
    return float(np.max(np.abs(Y_gpu_bf16.astype(np.float64) - ref_b) / ulp))
