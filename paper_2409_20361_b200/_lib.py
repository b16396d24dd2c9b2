"""ctypes binding of librrs.so (include/rrs.h).  Argument marshalling only: every step of the RRS
path runs in the CUDA kernels behind the C-ABI; there is no CPU or PyTorch fallback.

Tensors are torch tensors on the current CUDA device (torch supplies device memory and streams);
bf16 data may be passed as torch.bfloat16 or as raw torch.int16/uint16 bit patterns.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "librrs.so")

RRS_OK = 0
RRS_BF16 = 0
RRS_F32 = 1
RRS_GEMM_PLAIN = 0x1
RRS_OPERAND_I8 = 0x2
RRS_TOKEN_SHARDED = 0x4
RRS_GEMM_SWIGLU = 0x8
RRS_GEMM_SUBCHANNEL = 0x10
RRS_W_PACKED4 = 0x20
RRS_NO_ROTATION = 0x40
RRS_PREROTATED = 0x80
RRS_NO_SMOOTH = 0x100

_c_i64, _c_i32, _c_u32, _c_p, _c_sz, _c_f = (ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p,
                                             ctypes.c_size_t, ctypes.c_float)

_SIGS = {
    "rrs_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "rrs_last_error": (ctypes.c_char_p, []),
    "rrs_version": (ctypes.c_int, []),
    "rrs_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32]),
    "rrs_workspace_bytes_comm": (_c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32]),
    "rrs_perm_from_channel_max": (ctypes.c_int, [_c_p, _c_i64, _c_p, _c_p]),
    "rrs_prepare_weights": (ctypes.c_int, [_c_p, _c_i32, _c_i64, _c_i64, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_u32,
                                           _c_p]),
    "rrs_rotate_smooth_quant": (ctypes.c_int, [_c_p, _c_i32, _c_i64, _c_i64, _c_i32, _c_p, _c_p, _c_p, _c_p,
                                               _c_p, _c_p, _c_p, _c_sz, _c_u32, _c_p]),
    "rrs_gemm": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_f, _c_u32,
                                _c_p, _c_i32, _c_i64, _c_p]),
    "rrs_linear": (ctypes.c_int, [_c_p, _c_i32, _c_i64, _c_i64, _c_i32, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_i32,
                                  _c_i64, _c_p, _c_p, _c_sz, _c_u32, _c_p]),
    "rrs_allgather_columns": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_p, _c_p, _c_sz, _c_p]),
    "rrs_comm_unique_id": (ctypes.c_int, [_c_p]),
    "rrs_comm_init": (ctypes.c_int, [ctypes.POINTER(_c_p), _c_i32, _c_i32, _c_p]),
    "rrs_comm_destroy": (ctypes.c_int, [_c_p]),
    "rrs_comm_world": (_c_i32, [_c_p]),
    "rrs_comm_rank": (_c_i32, [_c_p]),
    "rrs_debug_rotate": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p]),
    "rrs_debug_group_partials": (ctypes.c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_p, _c_u32, _c_p]),
    "rrs_debug_relayout": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_p]),
}
EXPORTS = tuple(_SIGS)

_lib = None


class RRSError(RuntimeError):
    def __init__(self, fn: str, status: int):
        detail = lib().rrs_last_error().decode(errors="replace")
        name = lib().rrs_status_str(status).decode()
        super().__init__(f"{fn} -> {name}: {detail}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load librrs.so (loudly: there is no fallback if the extension is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() or "
                              "python -m paper_2409_20361_b200.build (no CPU fallback exists)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _ptr(t, row_strided: bool = False) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("librrs takes device tensors (got a CPU tensor)")
    ok = (t.dim() == 2 and t.stride(1) == 1) if row_strided else t.is_contiguous()
    if not ok:
        raise ValueError("librrs takes contiguous tensors (Y: unit column stride)")
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(fn: str, status: int) -> None:
    if status != RRS_OK:
        raise RRSError(fn, status)


def _bf16_code(t) -> int:
    if t.dtype in (torch.bfloat16, torch.int16, torch.uint16):
        return RRS_BF16
    raise TypeError(f"expected bf16 data (torch.bfloat16 or raw int16/uint16 bits), got {t.dtype}")


def _y_code(t) -> int:
    if t.dtype == torch.float32:
        return RRS_F32
    if t.dtype == torch.bfloat16:
        return RRS_BF16
    raise TypeError(f"Y must be float32 or bfloat16, got {t.dtype}")


# ------------------------------------------------------------------------- same names as include/rrs.h

def rrs_version() -> int:
    return lib().rrs_version()


def rrs_workspace_bytes(T: int, N: int, K: int, group: int = 128, world: int = 1) -> int:
    return int(lib().rrs_workspace_bytes(T, N, K, group, world))


def rrs_workspace_bytes_comm(T: int, N: int, K: int, group: int = 128, world: int = 1) -> int:
    """Workspace for rrs_linear with a communicator of `world` ranks (shard + all-gather buffers included)."""
    return int(lib().rrs_workspace_bytes_comm(T, N, K, group, world))


def rrs_perm_from_channel_max(chan_max, perm, stream=None) -> None:
    _check("rrs_perm_from_channel_max",
           lib().rrs_perm_from_channel_max(_ptr(chan_max), chan_max.numel(), _ptr(perm), _stream(stream)))


def _op_flags(i8: bool) -> int:
    return RRS_OPERAND_I8 if i8 else 0


def rrs_prepare_weights(W, perm, Wq, Wop, w_scale, group: int = 128, i8: bool = False, packed4: bool = False,
                        no_rotation: bool = False, stream=None) -> None:
    """Wop: uint8 [N][K] GEMM operand bytes (E4M3-encoded codes, or int8 codes with i8=True); with packed4=True
    Wop is the decode4 tiled nibble layout, ceil(N/256)*256 x K/2 bytes (RRS_W_PACKED4)."""
    N, K = W.shape
    _check("rrs_prepare_weights",
           lib().rrs_prepare_weights(_ptr(W), _bf16_code(W), N, K, group, _ptr(perm), _ptr(Wq), _ptr(Wop),
                                     _ptr(w_scale), _op_flags(i8) | (RRS_W_PACKED4 if packed4 else 0)
                                     | (RRS_NO_ROTATION if no_rotation else 0), _stream(stream)))


def _variant_flags(no_rotation: bool, prerotated: bool, no_smooth: bool) -> int:
    return ((RRS_NO_ROTATION if no_rotation else 0) | (RRS_PREROTATED if prerotated else 0)
            | (RRS_NO_SMOOTH if no_smooth else 0))


def rrs_rotate_smooth_quant(X, perm, Xq, Xop, x_scale, s_group, chan_max=None, ws=None, group: int = 128,
                            i8: bool = False, no_rotation: bool = False, prerotated: bool = False,
                            no_smooth: bool = False, stream=None) -> None:
    T, K = X.shape
    if ws is None:  # marshalling convenience: torch owns the scratch (X~ f32 + chan_max), see rrs_workspace_bytes
        ws = torch.empty(rrs_workspace_bytes(T, 1, K, group, 1), dtype=torch.uint8, device=X.device)
    _check("rrs_rotate_smooth_quant",
           lib().rrs_rotate_smooth_quant(_ptr(X), _bf16_code(X), T, K, group, _ptr(perm), _ptr(Xq), _ptr(Xop),
                                         _ptr(x_scale), _ptr(s_group), _ptr(chan_max), _ptr(ws),
                                         0 if ws is None else ws.numel() * ws.element_size(),
                                         _op_flags(i8) | _variant_flags(no_rotation, prerotated, no_smooth),
                                         _stream(stream)))


def rrs_gemm(Xop, x_scale, s_group, Wop, w_scale, Y, out_scale: float, plain: bool = False, group: int = 128,
             i8: bool = False, swiglu: bool = False, subchannel: bool = False, packed4: bool = False,
             stream=None) -> None:
    """subchannel: x_scale f32 [G][T], w_scale f32 [G][N] (the sub-channel A4W4 baseline), s_group unused.
    packed4: decode regime -- Xop int8 codes [T][K], Wop decode4-packed (RRS_W_PACKED4; N is then Y's width)."""
    T, K = Xop.shape
    N = Y.shape[1] * (2 if swiglu else 1) if packed4 else Wop.shape[0]
    flags = (RRS_GEMM_PLAIN if plain else 0) | _op_flags(i8) | (RRS_GEMM_SWIGLU if swiglu else 0) \
        | (RRS_GEMM_SUBCHANNEL if subchannel else 0) | (RRS_W_PACKED4 if packed4 else 0)
    _check("rrs_gemm",
           lib().rrs_gemm(_ptr(Xop), _ptr(x_scale), _ptr(s_group), _ptr(Wop), _ptr(w_scale), T, N, K, group,
                          float(out_scale), flags, _ptr(Y, True), _y_code(Y), Y.stride(0), _stream(stream)))


def rrs_linear(X, perm, Wop, w_scale, Y, ws, N_total: int | None = None, comm=None, group: int = 128,
               i8: bool = False, token_sharded: bool = False, swiglu: bool = False, packed4: bool = False,
               no_rotation: bool = False, prerotated: bool = False, no_smooth: bool = False, stream=None) -> None:
    T, K = X.shape
    N_total = (Y.shape[1] * (2 if swiglu else 1)) if N_total is None else N_total
    _check("rrs_linear",
           lib().rrs_linear(_ptr(X), _bf16_code(X), T, K, group, _ptr(perm), _ptr(Wop), _ptr(w_scale), N_total,
                            _ptr(Y, True), _y_code(Y), Y.stride(0), comm, _ptr(ws), ws.numel() * ws.element_size(),
                            _op_flags(i8) | (RRS_TOKEN_SHARDED if token_sharded else 0)
                            | (RRS_GEMM_SWIGLU if swiglu else 0) | (RRS_W_PACKED4 if packed4 else 0)
                            | _variant_flags(no_rotation, prerotated, no_smooth), _stream(stream)))


def rrs_allgather_columns(Y_shard, Y, comm, ws, stream=None) -> None:
    T = Y_shard.shape[0]
    N_total = Y.shape[1]
    _check("rrs_allgather_columns",
           lib().rrs_allgather_columns(_ptr(Y_shard), T, N_total, _y_code(Y_shard), _ptr(Y, True), Y.stride(0), comm,
                                       _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def rrs_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check("rrs_comm_unique_id", lib().rrs_comm_unique_id(buf))
    return bytes(buf)


def rrs_comm_init(rank: int, world: int, uid: bytes):
    h = _c_p()
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check("rrs_comm_init", lib().rrs_comm_init(ctypes.byref(h), rank, world, buf))
    return h.value


def rrs_comm_destroy(comm) -> None:
    _check("rrs_comm_destroy", lib().rrs_comm_destroy(comm))


def rrs_debug_rotate(X, Xr, chan_max, stream=None) -> None:
    T, K = X.shape
    _check("rrs_debug_rotate", lib().rrs_debug_rotate(_ptr(X), T, K, _ptr(Xr), _ptr(chan_max), _stream(stream)))


def rrs_debug_group_partials(Xop, Wop, P, group: int = 128, i8: bool = False, stream=None) -> None:
    T, K = Xop.shape
    N = Wop.shape[0]
    _check("rrs_debug_group_partials",
           lib().rrs_debug_group_partials(_ptr(Xop), _ptr(Wop), T, N, K, group, _ptr(P), _op_flags(i8),
                                          _stream(stream)))


def rrs_debug_relayout(gathered, Y, stream=None) -> None:
    """gathered: [world][T][n_shard] (f32 or bf16) -> Y[T][world * n_shard] (unit column stride, any row stride)."""
    world, T, ns = gathered.shape
    _check("rrs_debug_relayout",
           lib().rrs_debug_relayout(_ptr(gathered), T, ns, world, _y_code(gathered), _ptr(Y, True), Y.stride(0),
                                    _stream(stream)))
