"""Small-shape workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every kernel family of
librrs once -- prefill prologues (rows kernel K=1024, fused K=256, two-kernel K=14336... at small T), decode prologue,
pair and single-CTA GEMMs (RRS / plain / SwiGLU / sub-channel / split-K), the decode packed-W GEMM, the variants,
offline weight preparation and the relayout.  Exits 0 when every call returns and the device is error-free.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_20361_b200 as rrs  # noqa: E402
from rrs_synth import make_activations, make_weights  # noqa: E402


def dev_bf16(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).cuda().view(torch.bfloat16)


def layer_case(T, K, N, decode=False, swiglu=False, **kw):
    X = dev_bf16(make_activations("mixed", T, K, 11, 12))
    W = dev_bf16(make_weights(N, K, 13))
    perm = rrs.calibrate_perm(dev_bf16(make_activations("mixed", 64, K, 11, 14)))
    layer = rrs.RRSLinear(W, perm, decode=decode, swiglu=swiglu, **kw)
    for dt in (torch.float32, torch.bfloat16) if not swiglu else (torch.bfloat16,):
        layer(X, out_dtype=dt)
    return layer, X, perm


def main():
    torch.cuda.set_device(0)
    layer_case(8, 256, 256)                    # C1: fused prologue (K = 256), single-CTA GEMM
    layer_case(300, 1024, 264)                 # rows prologue (K = 1024), pair GEMM, ragged T and N
    layer_case(130, 14336, 256)                # two-kernel prologue (K = 28 * 512)
    layer_case(70, 4096, 256)                  # fused prologue on the 64-double plan (K = 4096), dynamic rows, ring
    layer_case(5, 8192, 512, decode=True)      # decode prologue + packed-W GEMM
    layer_case(1, 8192, 512, decode=True)      # decode prologue without a barrier (T = 1)
    layer_case(40, 2048, 512)                  # decode-sized T through the split-K GEMM
    layer_case(260, 2048, 496, swiglu=True)    # fused SwiGLU epilogue
    layer_case(130, 1024, 256, i8=True)        # int8 carrier
    T, K, N = 70, 1024, 256
    X = dev_bf16(make_activations("channel", T, K, 21, 22))
    perm = torch.arange(K, dtype=torch.int32, device="cuda")
    Xop = torch.empty((T, K), dtype=torch.uint8, device="cuda")
    xs, sg = torch.empty(T, device="cuda"), torch.empty(K // 128, device="cuda")
    for kw in ({"no_rotation": True}, {"prerotated": True}, {"no_smooth": True}):
        rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg, **kw)
    W = make_weights(N, K, 23)
    layer = rrs.RRSLinear(dev_bf16(W), perm)
    Y = torch.empty((T, N), device="cuda")
    rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg)
    rrs.rrs_gemm(Xop, xs, None, layer.Wop, layer.w_scale, Y, 1.0 / K, plain=True)
    G = K // 128
    rrs.rrs_gemm(Xop, torch.rand(G, T, device="cuda"), None, layer.Wop, torch.rand(G, N, device="cuda"), Y, 1.0 / K,
                 subchannel=True)
    g = torch.randn(3, 37, 24, device="cuda")
    rrs.rrs_debug_relayout(g, torch.empty(37, 72, device="cuda"))
    torch.cuda.synchronize()
    print("sanitize workload OK")


if __name__ == "__main__":
    main()
