"""Column-parallel layer on one GPU and, where the box has them, on two.

T3a: P in {2, 4, 8} ranks are emulated on one GPU with the product kernels -- each "rank" runs the RRS
GEMM on its W rows [r N/P, (r+1) N/P) (identical prologue codes: the prologue does not depend on W), the shards are
stacked rank-major exactly as ncclAllGather leaves them, and the product's relayout kernel (rrs_debug_relayout)
builds Y.  The result must equal the single-GPU layer BIT FOR BIT (output columns are independent: no reduction is
split), in f32, bf16 and with the fused SwiGLU epilogue (each rank holding whole gate/up pairs).

The torchrun world-2 test runs the real NCCL path on 2 GPUs (skipped on a 1-GPU box).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2409_20361_b200 as rrs  # noqa: E402
from oracle import rrs_oracle as o  # noqa: E402
from rrs_synth import bf16_bits_to_f64, make_activations, make_weights  # noqa: E402

from _parity import dev_bf16  # noqa: E402

DEV = "cuda"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _setup(T, N, K, seed):
    X_bits = make_activations("channel", T, K, 4000 + seed, 4001 + seed)
    W_bits = make_weights(N, K, 4002 + seed)
    perm = o.calibrate_perm(bf16_bits_to_f64(make_activations("channel", 64, K, 4000 + seed, 4003))).astype(np.int32)
    return dev_bf16(X_bits), dev_bf16(W_bits), torch.from_numpy(perm).to(DEV)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("out", ["f32", "bf16", "swiglu"])
def test_emulated_ranks_equal_single_gpu_bitwise(P, out):
    T, K = 1100, 2048
    N = 1920 if out != "swiglu" else 2 * 1920  # N/P a multiple of 16 bytes of output for every P
    X, W, perm = _setup(T, N, K, P)
    swiglu = out == "swiglu"
    if swiglu:
        W = rrs.interleave_gate_up(W[: N // 2], W[N // 2:])
    dt = torch.float32 if out == "f32" else torch.bfloat16
    full = rrs.RRSLinear(W, perm, swiglu=swiglu)
    Y1 = full(X, out_dtype=dt)
    # the prologue codes every rank computes (identical on every rank: they do not depend on W)
    Xop = torch.empty((T, K), dtype=torch.uint8, device=DEV)
    xs = torch.empty(T, dtype=torch.float32, device=DEV)
    sg = torch.empty(K // 128, dtype=torch.float32, device=DEV)
    rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg)
    ns = N // P
    n_out = ns // 2 if swiglu else ns
    gathered = torch.empty((P, T, n_out), dtype=dt, device=DEV)
    for r in range(P):
        lo, hi = rrs.shard_rows(N, P, r)
        shard = rrs.RRSLinear(W[lo:hi].contiguous(), perm, swiglu=swiglu)  # rank r's offline weight preparation
        assert torch.equal(shard.Wop, full.Wop[lo:hi]) and torch.equal(shard.w_scale, full.w_scale[lo:hi])
        rrs.rrs_gemm(Xop, xs, sg, shard.Wop, shard.w_scale, gathered[r], 1.0 / K, swiglu=swiglu)
    Y = torch.full_like(Y1, float("nan"))
    rrs.rrs_debug_relayout(gathered, Y)
    torch.cuda.synchronize()
    assert torch.equal(Y, Y1)


def test_relayout_ragged_row_stride():
    """Y a column block of a wider buffer (ldy > world * n_shard): columns outside stay untouched."""
    P, T, ns = 3, 37, 24
    g = torch.arange(P * T * ns, dtype=torch.float32, device=DEV).reshape(P, T, ns)
    Yb = torch.full((T, P * ns + 8), -1.0, device=DEV)
    rrs.rrs_debug_relayout(g, Yb[:, : P * ns])
    torch.cuda.synchronize()
    exp = g.permute(1, 0, 2).reshape(T, P * ns)
    assert torch.equal(Yb[:, : P * ns], exp) and bool((Yb[:, P * ns:] == -1).all())


_WORLD2 = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import numpy as np
import paper_2409_20361_b200 as rrs
from rrs_synth import make_activations, make_weights
from _parity import dev_bf16
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
comm = rrs.make_comm()[0]
T, N, K = 2048, 4096, 4096
X = dev_bf16(make_activations("channel", T, K, 7, 8), "cuda")
W = dev_bf16(make_weights(N, K, 9), "cuda")
perm = torch.arange(K, dtype=torch.int32, device="cuda")
Y1 = rrs.RRSLinear(W, perm)(X, out_dtype=torch.bfloat16)         # single-GPU layer on every rank
Yp = rrs.RRSLinear(W, perm, comm=comm, world=world, rank=rank)(X, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
ok = torch.tensor([int(torch.equal(Y1, Yp))], device="cuda")
dist.all_reduce(ok, op=dist.ReduceOp.MIN)
if rank == 0:
    print("WORLD2_OK" if ok.item() == 1 else "WORLD2_MISMATCH")
dist.destroy_process_group()
"""


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (this box has fewer)")
def test_torchrun_world2_column_parallel_bitwise(tmp_path):
    script = tmp_path / "world2.py"
    script.write_text(_WORLD2.format(root=ROOT))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29517", str(script)],
                       capture_output=True, text=True, timeout=600)
    assert "WORLD2_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
