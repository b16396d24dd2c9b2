"""Prologue timing (CUDA events, L2 flushed before each call) at the bench shapes, with the achieved FP64 DADD rate
and algorithmic HBM bytes.

    python tools/time_prologue.py [workload ...]
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


def main():
    names = sys.argv[1:] or ["c2_llama2_7b_qo", "c3_llama3_8b_up", "c5_llama3_70b_up_rank8", "c3_llama3_8b_down",
                             "c4_decode_t64", "c4_decode_t1"]
    flush = L2Flush("cuda")
    for name in names:
        w = WORKLOADS[name]
        X_bits, _, Xc = make_layer(w, index=list(WORKLOADS).index(name), N=8)
        X = dev_bf16(X_bits)
        perm = rrs.calibrate_perm(dev_bf16(Xc))
        T, K = w.T, w.K
        outs = {}
        res = {}
        for mode in ("fused", "two_kernel"):  # no chan_max output (the rrs_linear hot path) / with chan_max
            Xop = torch.empty((T, K), dtype=torch.uint8, device="cuda")
            xs = torch.empty(T, device="cuda")
            sg = torch.empty(K // 128, device="cuda")
            cm = torch.empty(K, device="cuda") if mode == "two_kernel" else None
            ws = torch.empty(rrs.rrs_workspace_bytes(T, 1, K, 128, 1), dtype=torch.uint8, device="cuda")
            ts = []
            for i in range(25):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg, chan_max=cm, ws=ws)
                b.record()
                if i >= 5:
                    ts.append((a, b))
            torch.cuda.synchronize()
            v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
            res[mode] = (statistics.median(v), v[0])
            outs[mode] = (Xop.clone(), xs.clone(), sg.clone())
        same = all(torch.equal(x, y) for x, y in zip(outs["fused"], outs["two_kernel"]))
        a_k = (K.bit_length() - 1) if K & (K - 1) == 0 else ((K // 28).bit_length() - 1 + 14)
        tnew = res["fused"][0] * 1e-6
        print(f"{name} T={T} K={K}: fused {res['fused'][0]:.2f} us (min {res['fused'][1]:.2f}), two-kernel "
              f"{res['two_kernel'][0]:.2f} us; outputs identical: {same}; fused: {T * K * a_k / tnew / 1e12:.2f} "
              f"T DADD/s, {T * (3 * K + 4) / tnew / 1e9:.0f} GB/s algorithmic", flush=True)

if __name__ == "__main__":
    main()
