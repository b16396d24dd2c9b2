"""B200-native Rotated Runtime Smooth (arXiv 2409.20361) A4W4 linear layer.

Public surface = the C-ABI of include/rrs.h, exposed with the same names by ._lib, plus two thin
conveniences that only allocate torch device memory and call those entry points:

  RRSLinear      offline weight preparation (rrs_prepare_weights) + forward (rrs_linear)
  make_comm      NCCL communicator for column-parallel layers; torch.distributed ferries the id
"""
from __future__ import annotations

import torch

from ._lib import (EXPORTS, RRSError, lib, rrs_allgather_columns, rrs_comm_destroy, rrs_comm_init, rrs_comm_unique_id,  # noqa: F401
                   rrs_debug_group_partials, rrs_debug_relayout, rrs_debug_rotate, rrs_gemm, rrs_linear, rrs_perm_from_channel_max,
                   rrs_prepare_weights, rrs_rotate_smooth_quant, rrs_version, rrs_workspace_bytes,
                   rrs_workspace_bytes_comm)

GROUP = 128


def shard_rows(N: int, world: int, rank: int) -> tuple[int, int]:
    """Output-feature range [lo, hi) of `rank` in the column-parallel layout."""
    if N % world:
        raise ValueError(f"N={N} not divisible by world={world}")
    n = N // world
    return rank * n, (rank + 1) * n


def calibrate_perm(X_cal: torch.Tensor, stream=None) -> torch.Tensor:
    """Offline reorder (R5): rotate the calibration activation, take its channel max, sort (GPU)."""
    T, K = X_cal.shape
    dev = X_cal.device
    Xr = torch.empty((T, K), dtype=torch.float32, device=dev)
    cm = torch.empty(K, dtype=torch.float32, device=dev)
    rrs_debug_rotate(X_cal, Xr, cm, stream=stream)
    perm = torch.empty(K, dtype=torch.int32, device=dev)
    rrs_perm_from_channel_max(cm, perm, stream=stream)
    return perm


class RRSLinear:
    """Y = RRS-A4W4(X) @ W^T for a bf16 nn.Linear weight W[N][K] (column shard when comm is given)."""

    def __init__(self, W: torch.Tensor, perm: torch.Tensor, comm=None, world: int = 1, rank: int = 0,
                 keep_packed: bool = False, i8: bool = False, group: int = GROUP, token_sharded: bool = False,
                 swiglu: bool = False, decode: bool = False, prerotated: bool = False, stream=None):
        """token_sharded: data parallel over tokens -- every rank keeps all N rows of W, calls
        with its own token slab and gets its own rows of Y; one all-reduce(MAX) of chan_max per call."""
        N, K = W.shape
        self.group = group  # smoothing group (128; any power of two in [32, 1024])
        self.K, self.N_total = K, N
        self.comm, self.world, self.rank = comm, world, rank
        self.token_sharded = token_sharded
        self.swiglu = swiglu  # rows are interleaved (gate_i, up_i) pairs; output = silu(gate) * up, N/2 columns
        # the input arrives already rotated (QuaRot-style rotation fused upstream): skip the online a1
        self.prerotated = prerotated
        lo, hi = (0, N) if token_sharded else shard_rows(N, world, rank)
        Wl = W[lo:hi].contiguous()
        dev = W.device
        self.perm = perm.to(device=dev, dtype=torch.int32).contiguous()
        self.i8 = i8  # GEMM operand carrier: E4M3 bytes (default) or int8 codes (RRS_OPERAND_I8)
        self.Wop = torch.empty((hi - lo, K), dtype=torch.uint8, device=dev)
        self.Wq = torch.empty((hi - lo, K // 2), dtype=torch.uint8, device=dev) if keep_packed else None
        self.w_scale = torch.empty(hi - lo, dtype=torch.float32, device=dev)
        rrs_prepare_weights(Wl, self.perm, self.Wq, self.Wop, self.w_scale, i8=i8, stream=stream)
        # decode regime (T <= 64, configs[3]): W also kept packed at 4 bits for the W-stream GEMM (RRS_W_PACKED4)
        self.Wp4 = None
        if decode and not swiglu and comm is None and group % 128 == 0:
            self.Wp4 = torch.empty(((hi - lo + 255) // 256 * 256, K // 2), dtype=torch.uint8, device=dev)
            rrs_prepare_weights(Wl, self.perm, None, self.Wp4, torch.empty_like(self.w_scale), packed4=True,
                                stream=stream)
        self._ws = None

    def workspace(self, T: int, device) -> torch.Tensor:
        if self.comm is not None and not self.token_sharded:  # column-parallel: shard + all-gather buffers
            need = rrs_workspace_bytes_comm(T, self.N_total, self.K, self.group, self.world)
        else:
            need = rrs_workspace_bytes(T, self.N_total, self.K, self.group, 1)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    def __call__(self, X: torch.Tensor, out_dtype=torch.bfloat16, Y: torch.Tensor | None = None, stream=None):
        T = X.shape[0]
        if Y is None:
            Y = torch.empty((T, self.N_total // (2 if self.swiglu else 1)), dtype=out_dtype, device=X.device)
        if self.Wp4 is not None and 1 <= T <= 64:
            rrs_linear(X, self.perm, self.Wp4, self.w_scale, Y, self.workspace(T, X.device), N_total=self.N_total,
                       group=self.group, packed4=True, prerotated=self.prerotated, stream=stream)
            return Y
        rrs_linear(X, self.perm, self.Wop, self.w_scale, Y, self.workspace(T, X.device), N_total=self.N_total,
                   comm=self.comm, group=self.group, i8=self.i8, token_sharded=self.token_sharded,
                   swiglu=self.swiglu, prerotated=self.prerotated, stream=stream)
        return Y


def interleave_gate_up(W_gate: torch.Tensor, W_up: torch.Tensor) -> torch.Tensor:
    """[F][K] gate and up weights -> [2F][K] with row 2i = gate_i, row 2i+1 = up_i (RRS_GEMM_SWIGLU layout)."""
    if W_gate.shape != W_up.shape:
        raise ValueError("gate / up shapes differ")
    return torch.stack([W_gate, W_up], dim=1).reshape(2 * W_gate.shape[0], W_gate.shape[1]).contiguous()


class RRSMLP:
    """LLaMA MLP block with RRS A4W4 linears (P:138 applies RRS to the up/gate and the down_proj
    inputs, where the paper places online rotation):
        h = silu(X W_gate^T) * (X W_up^T)   -- ONE prologue on X and ONE GEMM over the interleaved 2F rows,
                                               SwiGLU fused into the GEMM epilogue (bf16 h written once)
        Y = RRS(h) W_down^T                 -- the down_proj RRS layer (K = F, e.g. 14336 = 28 * 512)
    perm_in / perm_mid: offline reorders of X and of h (calibrate_perm on calibration activations)."""

    def __init__(self, W_gate, W_up, W_down, perm_in, perm_mid, i8: bool = False, prerotated_input: bool = False,
                 stream=None):
        """prerotated_input: X arrives already rotated (the paper rotates online only before the output and
        down projectors; the up/gate input carries the rotation fused into the residual stream)."""
        self.up_gate = RRSLinear(interleave_gate_up(W_gate, W_up), perm_in, i8=i8, swiglu=True,
                                 prerotated=prerotated_input, stream=stream)
        self.down = RRSLinear(W_down, perm_mid, i8=i8, stream=stream)

    def __call__(self, X: torch.Tensor, out_dtype=torch.bfloat16, stream=None):
        h = self.up_gate(X, out_dtype=torch.bfloat16, stream=stream)
        return self.down(h, out_dtype=out_dtype, stream=stream)


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL id (rrs_comm_unique_id); torch.distributed ferries it to every rank."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    uid = [rrs_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    if not isinstance(uid[0], bytes) or len(uid[0]) != 128:
        raise RuntimeError("NCCL unique id broadcast failed")
    return uid[0]


def make_comm(group=None):
    """NCCL communicator over the ranks of a torch.distributed group (rank 0's id is broadcast)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    return rrs_comm_init(rank, world, broadcast_unique_id(group)), rank, world
