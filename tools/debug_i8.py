"""Diagnose the i8-carrier bf16 mismatch: compare carriers bitwise and locate >1-ulp elements."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2409_20361_b200 as rrs
from oracle import rrs_oracle as o
from rrs_synth import WORKLOADS, bf16_bits_to_f64, make_layer
from _parity import dev_bf16, oracle_layer, y_normalised_error, bf16_ulp_error

w = WORKLOADS["c2_llama2_7b_qo"]
X_bits, W_bits, Xc = make_layer(w, T=300, N=264, T_cal=64)
perm = o.calibrate_perm(bf16_bits_to_f64(Xc)).astype(np.int32)
ref = oracle_layer(X_bits, W_bits, perm)
p = torch.from_numpy(perm).cuda()
res = {}
for i8 in (False, True):
    layer = rrs.RRSLinear(dev_bf16(W_bits), p, i8=i8)
    X = dev_bf16(X_bits)
    for rep in range(3):
        Yf = layer(X, out_dtype=torch.float32)
        Yb = layer(X, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        res[(i8, rep)] = (Yf.cpu().numpy(), Yb.float().cpu().numpy())
        print(f"i8={i8} rep={rep} f32 norm err {y_normalised_error(res[(i8,rep)][0], ref):.3e}  bf16 ulp err {bf16_ulp_error(res[(i8,rep)][1], ref['Y']):.2f}")
for rep in range(3):
    a, b = res[(False, rep)], res[(True, rep)]
    print("carrier f32 identical:", np.array_equal(a[0], b[0]), " bf16 identical:", np.array_equal(a[1], b[1]))
Yb = res[(True, 0)][1]
refb = o.bf16_round(ref["Y"])
m, e = np.frexp(np.where(refb == 0, 1.0, refb))
ulp = np.ldexp(1.0, e - 8)
err = np.abs(Yb - refb) / ulp
idx = np.argwhere(err > 1)
print("elements >1ulp:", len(idx), idx[:10].tolist())
for t, n in idx[:5]:
    print(t, n, "gpu bf16", Yb[t, n], "gpu f32", res[(True, 0)][0][t, n], "fp8 f32", res[(False, 0)][0][t, n], "ref", ref["Y"][t, n])
