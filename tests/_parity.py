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


def oracle_layer(X_bits, W_bits, perm, keep_partials=True, group=128):
    return o.rrs_linear(bf16_bits_to_f64(X_bits), bf16_bits_to_f64(W_bits), np.asarray(perm), L=group,
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


def bf16_ulp_error(Y_gpu_bf16: np.ndarray, Y_ref: np.ndarray, ref: dict | None = None) -> float:
    """|Y_gpu - bf16(Y_or)| in units of bf16 ulp of Y_or (DESIGN.md §5 bf16 reading).

    With `ref` (the oracle dict), the FP32 accumulation tolerance of R18 is granted on top: an element whose
    exact value sits within 1e-5 * alpha beta sum_g s_g |P_g| / K of a bf16 rounding boundary may round either
    way, so the allowance is (1e-5 * den) / ulp extra ulps (zero unless the element cancels)."""
    ref_b = o.bf16_round(Y_ref)
    m, e = np.frexp(np.where(ref_b == 0, 1.0, ref_b))
    ulp = np.ldexp(1.0, e - 8)
    err = np.abs(Y_gpu_bf16.astype(np.float64) - ref_b) / ulp
    if ref is not None:
        P = ref["P"].astype(np.float64)
        den = np.tensordot(ref["s_group"].astype(np.float64), np.abs(P), axes=(0, 0))
        den = den * ref["alpha"].astype(np.float64)[:, None] * ref["beta"].astype(np.float64)[None, :] * ref["out_scale"]
        err = err - (1e-5 * den) / ulp
    return float(np.max(err))


# ---- GEMM operand carriers (include/rrs.h): int8 codes, or E4M3 bytes.  The E4M3 table is built here from
# the format's definition (sign | 4-bit exponent, bias 7 | 3-bit fraction), independently of the product.
def _e4m3_value(b: int) -> float:
    s = -1.0 if b & 0x80 else 1.0
    e, m = (b >> 3) & 0xF, b & 7
    if e == 0xF and m == 7:
        return float("nan")
    return s * (m / 8.0) * 2.0 ** -6 if e == 0 else s * (1.0 + m / 8.0) * 2.0 ** (e - 7)


_E4M3_OF_INT = {}
for _b in range(256):
    _v = _e4m3_value(_b)
    if _v == _v and _v == int(_v) and -8 <= _v <= 7 and not (_v == 0 and _b != 0):
        _E4M3_OF_INT[int(_v)] = _b
_E4M3_LUT = np.array([_E4M3_OF_INT[q] for q in range(-8, 8)], dtype=np.uint8)
_E4M3_DEC = np.zeros(256, dtype=np.int16)
for _q, _b in _E4M3_OF_INT.items():
    _E4M3_DEC[_b] = _q


def encode_operand(q: np.ndarray, i8: bool) -> np.ndarray:
    """INT4 codes (int) -> GEMM operand bytes (uint8) for the chosen carrier."""
    q = np.asarray(q)
    return q.astype(np.int8).view(np.uint8) if i8 else _E4M3_LUT[q.astype(np.int64) + 8]


def decode_operand(b: np.ndarray, i8: bool) -> np.ndarray:
    """GEMM operand bytes -> INT4 codes (int8)."""
    b = np.asarray(b, dtype=np.uint8)
    return b.view(np.int8) if i8 else _E4M3_DEC[b].astype(np.int8)
