"""Quick timing of the decode regime (configs[3]) pieces with CUDA events, L2 flushed before each step.

    python tools/time_decode.py [T ...]
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_20361_b200 as rrs  # noqa: E402
from rrs_synth import WORKLOADS, make_layer  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench"))
from l2flush import L2Flush  # noqa: E402  (bench/l2flush.py)


def dev_bf16(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).cuda().view(torch.bfloat16)


def timeit(fn, flush, reps=30, warm=5):
    ts = []
    for i in range(warm + reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        if i >= warm:
            ts.append((a, b))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
    return statistics.median(v), v[0]


def main():
    Ts = [int(a) for a in sys.argv[1:]] or [1, 64]
    w = WORKLOADS["c4_decode_t64"]
    X_bits, W_bits, Xc = make_layer(w, index=list(WORKLOADS).index("c4_decode_t64"))
    perm = rrs.calibrate_perm(dev_bf16(Xc))
    layer = rrs.RRSLinear(dev_bf16(W_bits), perm, decode=True)
    flush = L2Flush("cuda")
    K, N = w.K, w.N
    for T in Ts:
        X = dev_bf16(X_bits[:T])
        Y = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
        ws = layer.workspace(T, "cuda")
        Xop = torch.empty((T, K), dtype=torch.uint8, device="cuda")
        xs = torch.empty(T, device="cuda")
        sg = torch.empty(K // 128, device="cuda")
        pws = torch.empty(rrs.rrs_workspace_bytes(T, 1, K, 128, 1), dtype=torch.uint8, device="cuda")
        res = {}
        res["layer_packed4"] = timeit(lambda: rrs.rrs_linear(X, perm, layer.Wp4, layer.w_scale, Y, ws, N_total=N,
                                                             packed4=True), flush)
        res["layer_bytes(r1)"] = timeit(lambda: rrs.rrs_linear(X, perm, layer.Wop, layer.w_scale, Y, ws, N_total=N),
                                        flush)
        res["prologue_i8"] = timeit(lambda: rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg, ws=pws, i8=True),
                                    flush)
        rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg, ws=pws, i8=True)
        res["decode_gemm"] = timeit(lambda: rrs.rrs_gemm(Xop, xs, sg, layer.Wp4, layer.w_scale, Y, 1.0 / K,
                                                         packed4=True), flush)
        # the same step replayed from a CUDA graph (how a serving loop launches decode steps)
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gs):
            for _ in range(3):
                rrs.rrs_linear(X, perm, layer.Wp4, layer.w_scale, Y, ws, N_total=N, packed4=True, stream=gs)
        torch.cuda.current_stream().wait_stream(gs)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            rrs.rrs_linear(X, perm, layer.Wp4, layer.w_scale, Y, ws, N_total=N, packed4=True, stream=gs)
        res["layer_packed4_graph"] = timeit(graph.replay, flush)
        gb = layer.Wp4.numel() / 1e9
        line = ", ".join(f"{k} {m:.2f} us (min {mn:.2f})" for k, (m, mn) in res.items())
        print(f"T={T}: {line}; decode GEMM W stream {gb / (res['decode_gemm'][0] * 1e-6):.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
