"""Prologue / layer variants of rrs.h (VERDICT r1 "next" 5) against the CPU oracle:

  RRS_NO_ROTATION  plain Runtime Smooth (Eq. 1-3): no Hadamard on X or W, out_scale 1
                   (oracle: rrs_linear(rotate_x=False))
  RRS_PREROTATED   X already rotated upstream (QuaRot-style): the prologue skips a1, W rotated offline,
                   out_scale 1/K (oracle: the rotated-W layer with the given X taken as X~)
  RRS_NO_SMOOTH    efficiency baselines only: s_g = 1 -> per-token RTN of X~ (QuaRot A4W4) or of X (plain A4W4)

Bar as everywhere: codes / alpha / s_g / chan_max bit-exact, Y within 1e-5 normalised error.  The
last test is the synthetic Table-4 trend measured through the GPU path.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2409_20361_b200 as rrs  # noqa: E402
from oracle import rrs_oracle as o  # noqa: E402
from rrs_synth import bf16_bits_to_f64, f64_to_bf16_bits, make_activations, make_weights  # noqa: E402

from _parity import decode_operand, dev_bf16, y_normalised_error  # noqa: E402

DEV = "cuda"


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _prologue(X_bits, perm, group=128, **kw):
    T, K = X_bits.shape
    Xq = torch.empty((T, K // 2), dtype=torch.uint8, device=DEV)
    Xop = torch.empty((T, K), dtype=torch.uint8, device=DEV)
    xs = torch.empty(T, dtype=torch.float32, device=DEV)
    sg = torch.empty(K // group, dtype=torch.float32, device=DEV)
    cm = torch.empty(K, dtype=torch.float32, device=DEV)
    rrs.rrs_rotate_smooth_quant(dev_bf16(X_bits), _dev(perm), Xq, Xop, xs, sg, chan_max=cm, group=group, **kw)
    torch.cuda.synchronize()
    return dict(Xq=Xq.cpu().numpy(), q=decode_operand(Xop.cpu().numpy(), False), alpha=xs.cpu().numpy(),
                s_group=sg.cpu().numpy(), chan_max=cm.cpu().numpy())


def _u(a):
    return np.asarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("K,T,profile,group", [(1024, 70, "spike", 128), (4096, 300, "channel", 64),
                                               (8192, 9, "mixed", 256), (14336, 40, "spike", 128)])
def test_no_rotation_prologue_bitexact(K, T, profile, group):
    """Plain Runtime Smooth: c_j = max_t |X_tj| on the UNROTATED activation, s_g, smooth, per-token RTN."""
    X_bits = make_activations(profile, T, K, 3100, 3101)
    perm = o.calibrate_perm(bf16_bits_to_f64(make_activations(profile, 64, K, 3100, 3102)), rotate_x=False)
    g = _prologue(X_bits, perm.astype(np.int32), group=group, no_rotation=True)
    Xr = bf16_bits_to_f64(X_bits).astype(np.float32)
    c = o.channel_max(Xr)
    s = o.group_scales(c, perm, group)
    q, a = o.smooth_quant(Xr, perm, s, group)
    assert np.array_equal(_u(g["chan_max"]), _u(c))
    assert np.array_equal(_u(g["s_group"]), _u(s))
    assert np.array_equal(_u(g["alpha"]), _u(a))
    assert np.array_equal(g["q"], q)
    assert np.array_equal(g["Xq"], o.pack_int4(q))


@pytest.mark.parametrize("rotate", [True, False], ids=["quarot", "plain"])
@pytest.mark.parametrize("K,T", [(4096, 129), (14336, 33), (8192, 5)])
def test_no_smooth_baseline_prologue(rotate, K, T):
    """RRS_NO_SMOOTH (the O_quarot / O_plain baselines of SURVEY §8(d)): s_g = 1, codes = per-token RTN of X~ (or X)."""
    X_bits = make_activations("channel", T, K, 3200, 3201)
    perm = np.arange(K, dtype=np.int32)[::-1].copy()
    g = _prologue(X_bits, perm, no_smooth=True, no_rotation=not rotate)
    X = bf16_bits_to_f64(X_bits)
    Xr = o.rotate(X) if rotate else X.astype(np.float32)
    q, a = o.quantize_rows(Xr[:, perm])
    assert np.all(g["s_group"] == 1.0)
    assert np.array_equal(_u(g["alpha"]), _u(a))
    assert np.array_equal(g["q"], q)


@pytest.mark.parametrize("K,T,N,profile", [(1024, 37, 264, "spike"), (4096, 300, 520, "channel"),
                                           (8192, 16, 256, "mixed")])
def test_no_rotation_layer(K, T, N, profile):
    """Whole plain-RS layer: W prepared without rotation (rrs_prepare_weights(RRS_NO_ROTATION)), out_scale 1."""
    X_bits = make_activations(profile, T, K, 3300, 3301)
    W_bits = make_weights(N, K, 3302)
    perm = o.calibrate_perm(bf16_bits_to_f64(make_activations(profile, 64, K, 3300, 3303)), rotate_x=False)
    ref = o.rrs_linear(bf16_bits_to_f64(X_bits), bf16_bits_to_f64(W_bits), perm, rotate_x=False)
    Wop = torch.empty((N, K), dtype=torch.uint8, device=DEV)
    Wq = torch.empty((N, K // 2), dtype=torch.uint8, device=DEV)
    ws = torch.empty(N, dtype=torch.float32, device=DEV)
    p = _dev(perm.astype(np.int32))
    rrs.rrs_prepare_weights(dev_bf16(W_bits), p, Wq, Wop, ws, no_rotation=True)
    Y = torch.empty((T, N), dtype=torch.float32, device=DEV)
    wsp = torch.empty(rrs.rrs_workspace_bytes(T, N, K, 128, 1), dtype=torch.uint8, device=DEV)
    rrs.rrs_linear(dev_bf16(X_bits), p, Wop, ws, Y, wsp, no_rotation=True)
    torch.cuda.synchronize()
    assert np.array_equal(Wq.cpu().numpy(), ref["Wq"])
    assert np.array_equal(_u(ws.cpu().numpy()), _u(ref["beta"]))
    assert y_normalised_error(Y.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("K,T,N", [(4096, 200, 264), (8192, 9, 520)])
def test_prerotated_layer(K, T, N):
    """RRS_PREROTATED (QKV / up / gate inputs are rotated upstream by the fused residual rotation): the caller
    passes X~ (bf16) directly, W is the usual rotated-offline weight, out_scale stays 1/K."""
    X_bits = make_activations("channel", T, K, 3400, 3401)
    W_bits = make_weights(N, K, 3402)
    # the upstream rotation: X~ = X H (rounded to the bf16 that the previous layer would emit)
    Xt_bits = f64_to_bf16_bits(o.rotate(bf16_bits_to_f64(X_bits)).astype(np.float64))
    perm = o.calibrate_perm(bf16_bits_to_f64(make_activations("channel", 64, K, 3400, 3403)))
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits), perm)  # rotated W (as for the online layer)
    ref = o.rrs_linear(bf16_bits_to_f64(Xt_bits), None, perm, rotate_x=False, prepared=(qw, beta))
    ref["out_scale"] = 1.0 / K
    ref["Y"] = ref["Y"] / K  # exact power-of-two rescale of the f64 result
    layer = rrs.RRSLinear(dev_bf16(W_bits), _dev(perm.astype(np.int32)))
    Y = torch.empty((T, N), dtype=torch.float32, device=DEV)
    rrs.rrs_linear(dev_bf16(Xt_bits), layer.perm, layer.Wop, layer.w_scale, Y, layer.workspace(T, DEV), prerotated=True)
    torch.cuda.synchronize()
    assert y_normalised_error(Y.cpu().numpy(), ref) <= 1e-5


def test_variant_flags_exclusive():
    K, T = 1024, 4
    X = torch.zeros((T, K), dtype=torch.bfloat16, device=DEV)
    p = torch.arange(K, dtype=torch.int32, device=DEV)
    Y = torch.empty((T, 64), device=DEV)
    ws = torch.empty(rrs.rrs_workspace_bytes(T, 64, K, 128, 1), dtype=torch.uint8, device=DEV)
    with pytest.raises(rrs.RRSError) as e:
        rrs.rrs_linear(X, p, torch.zeros((64, K), dtype=torch.uint8, device=DEV), torch.ones(64, device=DEV), Y, ws,
                       no_rotation=True, prerotated=True)
    assert e.value.status == 1


def test_table4_trend_through_gpu_path():
    """Synthetic Table 4 ("the accuracy deteriorates as the group size increases" for RS; RRS is
    "robust to the coarse group scheme"): relative Frobenius error of Y against the exact X W^T, through the GPU
    path at every group the kernels take (32 .. 512), channel-outlier profile.  RS (RRS_NO_ROTATION) error must grow
    with the group size; RRS stays within 15 % of its best.  Sanity of the method, not parity."""
    K, T, N = 1024, 256, 256
    X_bits = make_activations("channel", T, K, 5, 6)
    W_bits = make_weights(N, K, 7)
    Xc = bf16_bits_to_f64(make_activations("channel", 128, K, 5, 8))
    ref = bf16_bits_to_f64(X_bits) @ bf16_bits_to_f64(W_bits).T
    e_rs, e_rrs = [], []
    for L in (32, 64, 128, 256, 512):
        for rot, errs in ((False, e_rs), (True, e_rrs)):
            perm = _dev(o.calibrate_perm(Xc, rotate_x=rot).astype(np.int32))
            Wop = torch.empty((N, K), dtype=torch.uint8, device=DEV)
            ws = torch.empty(N, dtype=torch.float32, device=DEV)
            rrs.rrs_prepare_weights(dev_bf16(W_bits), perm, None, Wop, ws, no_rotation=not rot)
            Y = torch.empty((T, N), dtype=torch.float32, device=DEV)
            wsp = torch.empty(rrs.rrs_workspace_bytes(T, N, K, L, 1), dtype=torch.uint8, device=DEV)
            rrs.rrs_linear(dev_bf16(X_bits), perm, Wop, ws, Y, wsp, group=L, no_rotation=not rot)
            torch.cuda.synchronize()
            errs.append(np.linalg.norm(Y.cpu().numpy() - ref) / np.linalg.norm(ref))
    assert all(b >= a * 0.99 for a, b in zip(e_rs, e_rs[1:])), e_rs
    assert e_rs[-1] > 1.5 * e_rs[0], e_rs
    assert max(e_rrs) < 1.15 * min(e_rrs), e_rrs
    assert e_rrs[-1] < e_rs[-1]
