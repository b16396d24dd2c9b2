"""Multi-process host logic of the column-parallel layer, world_size 2 over gloo on CPU.

The GPU collective itself (ncclAllGather + relayout) needs GPUs; here we check what runs on the host and the
sharding invariant the column-parallel design relies on:
  * the NCCL unique id created by rank 0 reaches every rank intact (torch.distributed only ferries it);
  * shard_rows() partitions the N output features exactly, in rank order;
  * column shards of the RRS layer are independent: each rank's oracle output on its W rows, all-gathered
    and laid out by rank, equals the unsharded oracle output bit for bit (every rank runs the identical
    prologue on the replicated X, so s_g, alpha_t and the codes are the same everywhere);
  * bench.py's job time is the max over ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2409_20361_b200 as rrs
        from oracle import rrs_oracle as o
        from rrs_synth import WORKLOADS, bf16_bits_to_f64, make_layer
        import bench

        out = {}
        # 1. NCCL id broadcast
        uid = rrs.broadcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        out["ids_equal"] = all(i == ids[0] for i in ids) and len(uid) == 128

        # 2. shard partition
        N = 520
        lo, hi = rrs.shard_rows(N, world, rank)
        spans = [None] * world
        dist.all_gather_object(spans, (lo, hi))
        out["spans"] = spans

        # 3. sharded oracle == unsharded oracle, bitwise
        w = WORKLOADS["c2_llama2_7b_qo"]
        X_bits, W_bits, Xc = make_layer(w, T=40, N=N, T_cal=64)
        X, W = bf16_bits_to_f64(X_bits), bf16_bits_to_f64(W_bits)
        perm = o.calibrate_perm(bf16_bits_to_f64(Xc))
        mine = o.rrs_linear(X, W[lo:hi], perm, L=128, keep_partials=False)
        parts = [torch.empty((40, N // world), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(mine["Y"])))
        Y = torch.cat(parts, dim=1).numpy()
        out["gathered"] = Y
        out["prologue"] = (mine["s_group"].tobytes(), mine["alpha"].tobytes(), mine["Xq"].tobytes())

        # 5. token-sharded data parallel: each rank rotates its own token slab, the channel
        #    maxima are combined by an all-reduce(MAX) (the only exchange), then each rank smooths, quantises
        #    and multiplies its own tokens against all of W
        T = 40
        lo_t, hi_t = rank * T // world, (rank + 1) * T // world
        Xr = o.rotate(X[lo_t:hi_t])
        c = torch.from_numpy(o.channel_max(Xr).copy())
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        c = c.numpy()
        s = o.group_scales(c, perm, 128)
        codes, alpha = o.smooth_quant(Xr, perm, s, 128)
        qw, beta, _ = o.prepare_weights(W, perm)
        Yt = o.scale_accumulate_rows(codes, qw, s, alpha, beta, 128, 1.0 / X.shape[1])
        out["dp"] = dict(rows=(lo_t, hi_t), chan_max=c, s=s, q=codes, alpha=alpha, Y=Yt)

        # 4. bench timing reduction
        out["max"] = bench.max_over_ranks([1.0 + rank, 3.0 + rank], torch.device("cpu"), world)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def dist_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_unique_id_broadcast(dist_results):
    assert all(r["ids_equal"] for r in dist_results.values())


def test_shard_rows_partition(dist_results):
    spans = dist_results[0]["spans"]
    assert spans == [(0, 260), (260, 520)]
    with pytest.raises(ValueError):
        import paper_2409_20361_b200 as rrs
        rrs.shard_rows(10, 3, 0)


def test_sharded_equals_unsharded_bitwise(dist_results):
    from oracle import rrs_oracle as o
    from rrs_synth import WORKLOADS, bf16_bits_to_f64, make_layer
    w = WORKLOADS["c2_llama2_7b_qo"]
    X_bits, W_bits, Xc = make_layer(w, T=40, N=520, T_cal=64)
    perm = o.calibrate_perm(bf16_bits_to_f64(Xc))
    full = o.rrs_linear(bf16_bits_to_f64(X_bits), bf16_bits_to_f64(W_bits), perm, L=128, keep_partials=False)
    for r in dist_results.values():
        assert np.array_equal(r["gathered"], full["Y"])
    # identical prologue on every rank (replicated X)
    assert dist_results[0]["prologue"] == dist_results[1]["prologue"]


def test_max_over_ranks(dist_results):
    assert dist_results[0]["max"] == dist_results[1]["max"] == 3.0


def test_token_sharded_equals_unsharded_bitwise(dist_results):
    """all-reduce(MAX) of the per-rank channel maxima reproduces the call-wide maximum of Eq. 1
    (R6), so s_g, every code, alpha_t and every Y row equal the single call on all tokens."""
    from oracle import rrs_oracle as o
    from rrs_synth import WORKLOADS, bf16_bits_to_f64, make_layer
    w = WORKLOADS["c2_llama2_7b_qo"]
    X_bits, W_bits, Xc = make_layer(w, T=40, N=520, T_cal=64)
    perm = o.calibrate_perm(bf16_bits_to_f64(Xc))
    full = o.rrs_linear(bf16_bits_to_f64(X_bits), bf16_bits_to_f64(W_bits), perm, L=128, keep_partials=False)
    for r in dist_results.values():
        d = r["dp"]
        lo, hi = d["rows"]
        assert np.array_equal(d["chan_max"].view(np.uint32), full["chan_max"].view(np.uint32))
        assert np.array_equal(d["s"].view(np.uint32), full["s_group"].view(np.uint32))
        assert np.array_equal(d["q"], full["q"][lo:hi])
        assert np.array_equal(d["alpha"].view(np.uint32), full["alpha"][lo:hi].view(np.uint32))
        assert np.array_equal(d["Y"], full["Y"][lo:hi])
    spans = sorted(r["dp"]["rows"] for r in dist_results.values())
    assert spans == [(0, 20), (20, 40)]
