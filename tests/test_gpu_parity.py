"""CUDA path vs the CPU oracle, element by element, through the C-ABI (paper_2409_20361_b200._lib).

Bar (BASELINE.json north_star): bit-exact on X~, chan_max, s_group, alpha_t, every code,
every packed byte, beta_n, Wq and every int32 group partial P_g; Y f32 within normalised error 1e-5;
Y bf16 within 1 bf16 ulp.  Sizes span several 128x256 GEMM tiles and ragged T / N tails.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2409_20361_b200 as rrs  # noqa: E402
from oracle import rrs_oracle as o  # noqa: E402
from rrs_synth import WORKLOADS, bf16_bits_to_f64, make_activations, make_layer, make_weights  # noqa: E402

from _parity import (bf16_ulp_error, decode_operand, dev_bf16, encode_operand, oracle_layer,  # noqa: E402
                     y_normalised_error)

DEV = "cuda"


def _perm(Xc_bits):
    return o.calibrate_perm(bf16_bits_to_f64(Xc_bits)).astype(np.int32)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _run_prologue(X_bits, perm, i8=False, group=128):
    T, K = X_bits.shape
    X = dev_bf16(X_bits)
    p = torch.from_numpy(perm).to(DEV)
    Xq = torch.empty((T, K // 2), dtype=torch.uint8, device=DEV)
    Xop = torch.empty((T, K), dtype=torch.uint8, device=DEV)
    xs = torch.empty(T, dtype=torch.float32, device=DEV)
    sg = torch.empty(K // group, dtype=torch.float32, device=DEV)
    cm = torch.empty(K, dtype=torch.float32, device=DEV)
    rrs.rrs_rotate_smooth_quant(X, p, Xq, Xop, xs, sg, chan_max=cm, group=group, i8=i8)
    # the operand-only call (Xq = NULL) is the rrs_linear hot path, which takes a separate code path in the
    # quantisation kernel: its bytes must be identical
    # (and, for prefill K = 2^m, the group-max fused prologue: no chan_max requested)
    Xop2, xs2, sg2 = torch.empty_like(Xop), torch.empty_like(xs), torch.empty_like(sg)
    rrs.rrs_rotate_smooth_quant(X, p, None, Xop2, xs2, sg2, group=group, i8=i8)
    torch.cuda.synchronize()
    assert torch.equal(Xop, Xop2)
    assert torch.equal(xs, xs2) and torch.equal(sg, sg2)
    return dict(Xq=Xq.cpu().numpy(), Xop=Xop.cpu().numpy(), Xq8=decode_operand(Xop.cpu().numpy(), i8),
                alpha=xs.cpu().numpy(), s_group=sg.cpu().numpy(), chan_max=cm.cpu().numpy())


def _run_weights(W_bits, perm, i8=False):
    N, K = W_bits.shape
    Wq = torch.empty((N, K // 2), dtype=torch.uint8, device=DEV)
    Wop = torch.empty((N, K), dtype=torch.uint8, device=DEV)
    ws = torch.empty(N, dtype=torch.float32, device=DEV)
    rrs.rrs_prepare_weights(dev_bf16(W_bits), torch.from_numpy(perm).to(DEV), Wq, Wop, ws, i8=i8)
    torch.cuda.synchronize()
    return Wq.cpu().numpy(), Wop, ws


# ------------------------------------------------------------------------------------- a1 / a2

@pytest.mark.parametrize("K,T,profile", [(128, 5, "channel"), (256, 37, "tiny"), (1024, 64, "spike"),
                                         (4096, 33, "channel"), (8192, 9, "mixed"), (16384, 3, "channel"),
                                         (7168, 11, "spike"), (14336, 13, "spike")])
def test_rotation_and_channel_max_bitexact(K, T, profile):
    X_bits = make_activations(profile, T, K, 101, 202)
    Xr = torch.empty((T, K), dtype=torch.float32, device=DEV)
    cm = torch.empty(K, dtype=torch.float32, device=DEV)
    rrs.rrs_debug_rotate(dev_bf16(X_bits), Xr, cm)
    torch.cuda.synchronize()
    ref = o.rotate(bf16_bits_to_f64(X_bits))
    assert np.array_equal(_u32(Xr), ref.view(np.uint32))
    assert np.array_equal(_u32(cm), o.channel_max(ref).view(np.uint32))


# ------------------------------------------------------------------------------------- a3-a6

@pytest.mark.parametrize("K,T,profile", [(256, 8, "tiny"), (256, 300, "channel"), (4096, 129, "channel"),
                                         (14336, 40, "spike"), (8192, 64, "mixed"), (512, 1, "channel")])
@pytest.mark.parametrize("i8", [False, True], ids=["e4m3", "i8"])
def test_prologue_bitexact(K, T, profile, i8):
    X_bits = make_activations(profile, T, K, 303, 404)
    perm = _perm(make_activations(profile, 64, K, 303, 405))
    g = _run_prologue(X_bits, perm, i8=i8)
    Xr = o.rotate(bf16_bits_to_f64(X_bits))
    c = o.channel_max(Xr)
    s = o.group_scales(c, perm, 128)
    q, a = o.smooth_quant(Xr, perm, s, 128)
    assert np.array_equal(g["chan_max"].view(np.uint32), c.view(np.uint32))
    assert np.array_equal(g["s_group"].view(np.uint32), s.view(np.uint32))
    assert np.array_equal(g["alpha"].view(np.uint32), a.view(np.uint32))
    assert np.array_equal(g["Xq8"], q)
    assert np.array_equal(g["Xop"], encode_operand(q, i8))  # every operand byte
    assert np.array_equal(g["Xq"], o.pack_int4(q))


@pytest.mark.parametrize("K,T,profile,group", [(1024, 70, "channel", 32), (4096, 129, "spike", 64),
                                               (4096, 40, "mixed", 256), (14336, 24, "channel", 512),
                                               (2048, 9, "channel", 1024), (256, 300, "channel", 32)])
def test_prologue_group_variants_bitexact(K, T, profile, group):
    """SURVEY §8 f3 / Table 4: the smoothing group is a parameter (P:189 picks 128)."""
    X_bits = make_activations(profile, T, K, 313, 414)
    perm = _perm(make_activations(profile, 64, K, 313, 415))
    g = _run_prologue(X_bits, perm, group=group)
    Xr = o.rotate(bf16_bits_to_f64(X_bits))
    s = o.group_scales(o.channel_max(Xr), perm, group)
    q, a = o.smooth_quant(Xr, perm, s, group)
    assert g["s_group"].shape == (K // group,)
    assert np.array_equal(g["s_group"].view(np.uint32), s.view(np.uint32))
    assert np.array_equal(g["alpha"].view(np.uint32), a.view(np.uint32))
    assert np.array_equal(g["Xq8"], q)
    assert np.array_equal(g["Xq"], o.pack_int4(q))


def test_prologue_zero_rows_and_identity_perm():
    """R8: all-zero tokens -> alpha 1, codes 0; zero channels make no group scale 0 unless the group is."""
    K, T = 512, 20
    X_bits = make_activations("channel", T, K, 1, 2)
    X_bits[[0, 7, 19]] = 0
    perm = np.arange(K, dtype=np.int32)
    g = _run_prologue(X_bits, perm)
    r = o.rrs_linear(bf16_bits_to_f64(X_bits), np.zeros((1, K)), perm, keep_partials=False)
    assert np.array_equal(g["alpha"].view(np.uint32), r["alpha"].view(np.uint32))
    assert np.all(g["alpha"][[0, 7, 19]] == 1.0) and not g["Xq8"][[0, 7, 19]].any()
    assert np.array_equal(g["Xq8"], r["q"])


def test_prologue_all_zero_activation():
    K, T = 256, 4
    g = _run_prologue(np.zeros((T, K), np.uint16), np.arange(K, dtype=np.int32))
    assert np.all(g["s_group"] == 1.0) and np.all(g["alpha"] == 1.0) and not g["Xq8"].any()


# ------------------------------------------------------------------------------------- a7

@pytest.mark.parametrize("K,N", [(256, 256), (4096, 300), (14336, 64)])
@pytest.mark.parametrize("i8", [False, True], ids=["e4m3", "i8"])
def test_prepare_weights_bitexact(K, N, i8):
    W_bits = make_weights(N, K, 77)
    perm = _perm(make_activations("channel", 64, K, 5, 6))
    Wq, Wop, ws = _run_weights(W_bits, perm, i8=i8)
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits), perm)
    assert np.array_equal(Wop.cpu().numpy(), encode_operand(qw, i8))
    assert np.array_equal(Wq, o.pack_int4(qw))
    assert np.array_equal(_u32(ws), beta.view(np.uint32))


# ------------------------------------------------------------------------------------- a8 / a9

@pytest.mark.parametrize("T,N,K", [(8, 256, 256), (300, 600, 512), (129, 257, 4096), (1, 16, 128), (256, 512, 1024),
                                   (520, 488, 2048)])
@pytest.mark.parametrize("i8", [False, True], ids=["e4m3", "i8"])
def test_group_partials_bitexact(T, N, K, i8):
    """P_g read back from TMEM equals the oracle's integer group sums exactly, for both carriers (the FP8
    carrier's FP32 accumulation is exact because every partial is an integer below 2^13)."""
    rng = np.random.default_rng(T * 7 + N)
    q = rng.integers(-7, 8, size=(T, K)).astype(np.int8)
    qw = rng.integers(-7, 8, size=(N, K)).astype(np.int8)
    q[0, :] = 7   # extreme partials: +-49 * 128
    qw[0, :] = -7
    if T > 1 and N > 1:
        q[1, :] = -7
        qw[1, ::2] = 7  # alternating signs: large cancellations inside a group
        qw[1, 1::2] = -7
    P = torch.empty((K // 128, T, N), dtype=torch.int32, device=DEV)
    rrs.rrs_debug_group_partials(_dev(encode_operand(q, i8)), _dev(encode_operand(qw, i8)), P, i8=i8)
    torch.cuda.synchronize()
    assert np.array_equal(P.cpu().numpy(), o.group_partials(q, qw, 128))


@pytest.mark.parametrize("T,N,K,group", [(300, 600, 512, 32), (129, 257, 1024, 64), (520, 488, 2048, 256),
                                         (64, 240, 4096, 512), (8, 256, 1024, 1024)])
@pytest.mark.parametrize("i8", [False, True], ids=["e4m3", "i8"])
def test_group_partials_group_variants_bitexact(T, N, K, group, i8):
    """Per-group partials for groups smaller than (closed inside) and larger than (spanning) a 128-deep K-block."""
    rng = np.random.default_rng(T * 11 + group)
    q = rng.integers(-7, 8, size=(T, K)).astype(np.int8)
    qw = rng.integers(-7, 8, size=(N, K)).astype(np.int8)
    q[0, :] = 7
    qw[0, :] = -7  # |P_g| = 49 * group, the extreme
    P = torch.empty((K // group, T, N), dtype=torch.int32, device=DEV)
    rrs.rrs_debug_group_partials(_dev(encode_operand(q, i8)), _dev(encode_operand(qw, i8)), P, group=group, i8=i8)
    torch.cuda.synchronize()
    assert np.array_equal(P.cpu().numpy(), o.group_partials(q, qw, group))


def _gemm_case(T, N, K, profile="channel", seed=0):
    X_bits = make_activations(profile, T, K, 900 + seed, 901 + seed)
    W_bits = make_weights(N, K, 902 + seed)
    perm = _perm(make_activations(profile, 64, K, 900 + seed, 903 + seed))
    ref = oracle_layer(X_bits, W_bits, perm)
    return X_bits, W_bits, perm, ref


@pytest.mark.parametrize("T,N,K,profile", [(8, 256, 256, "tiny"), (300, 600, 512, "channel"),
                                           (129, 520, 4096, "channel"), (200, 264, 14336, "spike"),
                                           (64, 512, 8192, "mixed")])
@pytest.mark.parametrize("i8", [False, True], ids=["e4m3", "i8"])
def test_rrs_gemm_y_f32_and_bf16(T, N, K, profile, i8):
    X_bits, W_bits, perm, ref = _gemm_case(T, N, K, profile)
    Xq8 = _dev(encode_operand(ref["q"], i8))
    Wq8 = _dev(encode_operand(ref["qw"], i8))
    xs = torch.from_numpy(ref["alpha"]).to(DEV)
    sg = torch.from_numpy(ref["s_group"]).to(DEV)
    ws = torch.from_numpy(ref["beta"]).to(DEV)
    ldy = (N + 7) // 8 * 8
    Yf = torch.full((T, ldy), float("nan"), dtype=torch.float32, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wq8, ws, Yf[:, :N], 1.0 / K, i8=i8)
    Yb = torch.full((T, ldy), float("nan"), dtype=torch.bfloat16, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wq8, ws, Yb[:, :N], 1.0 / K, i8=i8)
    torch.cuda.synchronize()
    Yf_np = Yf.cpu().numpy()
    assert np.isnan(Yf_np[:, N:]).all()  # nothing written past N
    assert torch.isnan(Yb[:, N:].float()).all()  # bf16 (TMA-stored when N % 8 == 0) too
    assert y_normalised_error(Yf_np[:, :N], ref) <= 1e-5
    assert bf16_ulp_error(Yb[:, :N].float().cpu().numpy(), ref["Y"], ref) <= 1.0
    # bf16 output is the round-to-nearest-even of the very same f32 accumulation
    assert torch.equal(Yb[:, :N], Yf[:, :N].to(torch.bfloat16))


@pytest.mark.parametrize("T", [130, 100])
@pytest.mark.parametrize("i8", [False, True], ids=["e4m3", "i8"])
def test_plain_gemm_matches_per_channel_baseline(T, i8):
    """RRS_GEMM_PLAIN: Y = alpha beta sum_all q qw / K (per-channel A4W4)."""
    X_bits, W_bits, perm, ref = _gemm_case(T, 300, 1024)
    Xq8 = _dev(encode_operand(ref["q"], i8))
    Wq8 = _dev(encode_operand(ref["qw"], i8))
    Y = torch.empty((T, 304), dtype=torch.float32, device=DEV)
    rrs.rrs_gemm(Xq8, torch.from_numpy(ref["alpha"]).to(DEV), None, Wq8, torch.from_numpy(ref["beta"]).to(DEV),
                 Y[:, :300], 1.0 / 1024, plain=True, i8=i8)
    torch.cuda.synchronize()
    Pall = ref["P"].astype(np.int64).sum(axis=0).astype(np.float64)
    exp = Pall * ref["alpha"].astype(np.float64)[:, None] * ref["beta"].astype(np.float64)[None, :] / 1024
    den = np.abs(ref["P"]).astype(np.float64).sum(0) * ref["alpha"][:, None] * ref["beta"][None, :] / 1024
    err = np.abs(Y[:, :300].cpu().numpy() - exp)
    assert np.all(err <= 1e-5 * np.maximum(den, 1e-30))


# ------------------------------------------------------------------------------------- whole layer

@pytest.mark.parametrize("wl,T,N,i8", [("c1_tiny", None, None, False), ("c2_llama2_7b_qo", 257, 520, False),
                                       ("c3_llama3_8b_down", 130, 264, False), ("c2_llama2_7b_qo", 300, 264, True),
                                       ("c1_tiny", None, None, True)])
def test_rrs_linear_end_to_end(wl, T, N, i8):
    w = WORKLOADS[wl]
    X_bits, W_bits, Xc = make_layer(w, T=T, N=N, T_cal=64)
    T, N = X_bits.shape[0], W_bits.shape[0]
    perm = _perm(Xc)
    ref = oracle_layer(X_bits, W_bits, perm)
    layer = rrs.RRSLinear(dev_bf16(W_bits), torch.from_numpy(perm).to(DEV), keep_packed=True, i8=i8)
    Y = layer(dev_bf16(X_bits), out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert np.array_equal(layer.Wq.cpu().numpy(), ref["Wq"])
    assert y_normalised_error(Y.cpu().numpy(), ref) <= 1e-5
    Yb = layer(dev_bf16(X_bits), out_dtype=torch.bfloat16)
    assert bf16_ulp_error(Yb.float().cpu().numpy(), ref["Y"], ref) <= 1.0
    assert torch.equal(Yb, Y.to(torch.bfloat16))  # RNE of the same f32 accumulation


@pytest.mark.parametrize("T,N,K,group,i8", [(257, 520, 4096, 32, False), (130, 264, 4096, 64, True),
                                            (300, 264, 14336, 256, False), (129, 240, 8192, 512, False),
                                            (64, 256, 2048, 1024, True)])
def test_rrs_linear_group_variants(T, N, K, group, i8):
    """Whole layer at the Table-4 group sizes: codes from the same seeded LLaMA-like inputs,
    Y within the DESIGN.md §5 tolerance of the oracle run with the same group."""
    X_bits = make_activations("mixed", T, K, 930, 931)
    W_bits = make_weights(N, K, 932)
    perm = _perm(make_activations("mixed", 64, K, 930, 933))
    ref = oracle_layer(X_bits, W_bits, perm, group=group)
    layer = rrs.RRSLinear(dev_bf16(W_bits), torch.from_numpy(perm).to(DEV), i8=i8, group=group)
    Y = layer(dev_bf16(X_bits), out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert y_normalised_error(Y.cpu().numpy(), ref) <= 1e-5


def test_swiglu_epilogue_tma_width():
    """F % 8 == 0, ragged T, Y a sub-block of a larger buffer: every output written, nothing outside it."""
    T, F, K = 300, 248, 2048
    X_bits, W_bits, perm, ref = _gemm_case(T, 2 * F, K, "channel", seed=8)
    Xq8 = _dev(encode_operand(ref["q"], False))
    Wq8 = _dev(encode_operand(ref["qw"], False))
    xs, sg, ws = (torch.from_numpy(ref[k]).to(DEV) for k in ("alpha", "s_group", "beta"))
    Yf = torch.empty((T, 2 * F), dtype=torch.float32, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wq8, ws, Yf, 1.0 / K)
    H = torch.full((T + 5, F + 8), float("nan"), dtype=torch.bfloat16, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wq8, ws, H[:T, :F], 1.0 / K, swiglu=True)
    torch.cuda.synchronize()
    Y = Yf.cpu().numpy().astype(np.float64)
    Hn = H.float().cpu().numpy()
    assert np.isnan(Hn[:, F:]).all() and np.isnan(Hn[T:]).all()
    assert bf16_ulp_error(Hn[:T, :F], o.swiglu(Y[:, 0::2], Y[:, 1::2])) <= 1.0


@pytest.mark.parametrize("T,N,K,out,i8", [(1, 1024, 8192, "f32", False), (17, 1024, 8192, "bf16", False),
                                          (64, 488, 8192, "f32", False), (100, 520, 14336, "f32", False),
                                          (128, 264, 4096, "bf16", False), (33, 512, 8192, "f32", True),
                                          (5, 264, 2048, "bf16", True)])
def test_decode_split_k(T, N, K, out, i8):
    """Decode-sized T (<= 128, configs[3]): rrs_linear splits K over up to 8 CTAs per output tile (whole groups
    each) and sums the f32 partials in a fixed order -- same bar against the oracle, deterministic."""
    X_bits, W_bits, perm, ref = _gemm_case(T, N, K, "mixed", seed=T)
    layer = rrs.RRSLinear(dev_bf16(W_bits), torch.from_numpy(perm).to(DEV), i8=i8)
    X = dev_bf16(X_bits)
    if out == "f32":
        Y = layer(X, out_dtype=torch.float32)
        Y2 = layer(X, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert torch.equal(Y, Y2)
        assert y_normalised_error(Y.cpu().numpy(), ref) <= 1e-5
    else:
        Y = layer(X, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        assert bf16_ulp_error(Y.float().cpu().numpy(), ref["Y"], ref) <= 1.0


@pytest.mark.parametrize("T,N,K,group,out", [(300, 520, 2048, 128, "f32"), (129, 488, 4096, 256, "bf16"),
                                             (64, 264, 1024, 64, "f32")])
def test_subchannel_gemm_baseline(T, N, K, group, out):
    """RRS_GEMM_SUBCHANNEL (SURVEY §8 f4, P:322's second efficiency baseline): per (token, group) and per
    (row, group) RTN scales; Y within the §5 bar of the oracle's sum_g alpha_gt beta_gn P_g (f64)."""
    X = bf16_bits_to_f64(make_activations("channel", T, K, 960, 961)).astype(np.float32)
    W = bf16_bits_to_f64(make_weights(N, K, 962)).astype(np.float32)
    q, a = o.subchannel_quant(X, group)
    qw, b = o.subchannel_quant(W, group)
    ref = o.subchannel_gemm(q, qw, a, b, group)
    P = o.group_partials(q, qw, group).astype(np.float64)
    den = np.einsum("gt,gn,gtn->tn", a.astype(np.float64), b.astype(np.float64), np.abs(P))
    Xq8, Wq8 = _dev(encode_operand(q, False)), _dev(encode_operand(qw, False))
    ta, tb = _dev(a), _dev(b)
    if out == "f32":
        Y = torch.full((T, N), float("nan"), dtype=torch.float32, device=DEV)
        rrs.rrs_gemm(Xq8, ta, None, Wq8, tb, Y, 1.0, group=group, subchannel=True)
        torch.cuda.synchronize()
        err = np.abs(Y.cpu().numpy().astype(np.float64) - ref)
        assert np.all(err <= 1e-5 * den + (den == 0) * 0.0)
    else:
        Y = torch.full((T, N), float("nan"), dtype=torch.bfloat16, device=DEV)
        rrs.rrs_gemm(Xq8, ta, None, Wq8, tb, Y, 1.0, group=group, subchannel=True)
        torch.cuda.synchronize()
        ref_b = o.bf16_round(ref)
        _, e = np.frexp(np.where(ref_b == 0, 1.0, ref_b))
        ulp = np.ldexp(1.0, e - 8)
        assert np.all(np.abs(Y.float().cpu().numpy().astype(np.float64) - ref_b) <= ulp + 1e-5 * den)


@pytest.mark.parametrize("i8", [False, True], ids=["e4m3", "i8"])
def test_swiglu_epilogue(i8):
    """RRS_GEMM_SWIGLU: with interleaved (gate, up) rows the bf16 output is, within 1 bf16 ulp,
    bf16(silu(y_2i) * y_2i+1) of the very same GEMM's f32 output (the epilogue math is f32: one f32 product with
    beta, e^-g and a division), and that f32 output meets the §5 bar against the oracle."""
    T, F, K = 257, 260, 4096
    X_bits, W_bits, perm, ref = _gemm_case(T, 2 * F, K, "mixed", seed=7)
    Xq8 = _dev(encode_operand(ref["q"], i8))
    Wq8 = _dev(encode_operand(ref["qw"], i8))
    xs, sg, ws = (torch.from_numpy(ref[k]).to(DEV) for k in ("alpha", "s_group", "beta"))
    Yf = torch.empty((T, 2 * F), dtype=torch.float32, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wq8, ws, Yf, 1.0 / K, i8=i8)
    H = torch.full((T, F + 4), float("nan"), dtype=torch.bfloat16, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wq8, ws, H[:, :F], 1.0 / K, swiglu=True, i8=i8)
    torch.cuda.synchronize()
    Y = Yf.cpu().numpy().astype(np.float64)
    assert y_normalised_error(Yf.cpu().numpy(), ref) <= 1e-5
    h_ref = o.swiglu(Y[:, 0::2], Y[:, 1::2])
    Hn = H.float().cpu().numpy()
    assert np.isnan(Hn[:, F:]).all()  # nothing written past N/2
    assert bf16_ulp_error(Hn[:, :F], h_ref) <= 1.0


def test_rrs_mlp_block():
    """LLaMA MLP with RRS on the up/gate input (one prologue, one GEMM over 2F interleaved rows,
    fused SwiGLU) and on the down_proj input (K = F = 7168 = 28 * 256, the 28*2^m rotation).  Stage by stage:
    up/gate f32 output vs the oracle, h vs bf16(swiglu(that output)), down output vs the oracle run on h."""
    T, D, F = 130, 1024, 7168
    X_bits = make_activations("channel", T, D, 950, 951)
    Xc_bits = make_activations("channel", 64, D, 950, 952)
    Wg, Wu, Wd = make_weights(F, D, 953), make_weights(F, D, 954), make_weights(D, F, 955)
    perm_in = _perm(Xc_bits)
    Wug = np.stack([Wg, Wu], axis=1).reshape(2 * F, D)
    # calibration of the down_proj reorder on the oracle's h of the calibration tokens
    cal = oracle_layer(Xc_bits, Wug, perm_in, keep_partials=False)
    h_cal = o.bf16_round(o.swiglu(cal["Y"][:, 0::2], cal["Y"][:, 1::2]))
    perm_mid = o.calibrate_perm(h_cal).astype(np.int32)
    mlp = rrs.RRSMLP(dev_bf16(Wg), dev_bf16(Wu), dev_bf16(Wd), torch.from_numpy(perm_in).to(DEV),
                     torch.from_numpy(perm_mid).to(DEV))
    X = dev_bf16(X_bits)
    Y = mlp(X, out_dtype=torch.float32)
    h = torch.full((T, F), float("nan"), dtype=torch.bfloat16, device=DEV)  # no stale allocator memory
    mlp.up_gate(X, Y=h)
    ug_f32 = rrs.RRSLinear(dev_bf16(Wug), torch.from_numpy(perm_in).to(DEV))(X, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref_ug = oracle_layer(X_bits, Wug, perm_in)
    assert y_normalised_error(ug_f32.cpu().numpy(), ref_ug) <= 1e-5
    Yug = ug_f32.cpu().numpy().astype(np.float64)
    assert bf16_ulp_error(h.float().cpu().numpy(), o.swiglu(Yug[:, 0::2], Yug[:, 1::2])) <= 1.0
    h_bits = h.view(torch.int16).cpu().numpy().view(np.uint16)
    ref_down = oracle_layer(h_bits, Wd, perm_mid)
    assert y_normalised_error(Y.cpu().numpy(), ref_down) <= 1e-5


def test_rrs_linear_equals_prologue_plus_gemm_bitwise():
    X_bits, W_bits, perm, ref = _gemm_case(200, 512, 4096)
    X = dev_bf16(X_bits)
    p = torch.from_numpy(perm).to(DEV)
    layer = rrs.RRSLinear(dev_bf16(W_bits), p)
    Y1 = layer(X, out_dtype=torch.float32)
    Xop = torch.empty((200, 4096), dtype=torch.uint8, device=DEV)
    xs = torch.empty(200, dtype=torch.float32, device=DEV)
    sg = torch.empty(32, dtype=torch.float32, device=DEV)
    ws = torch.empty(rrs.rrs_workspace_bytes(200, 512, 4096), dtype=torch.uint8, device=DEV)
    rrs.rrs_rotate_smooth_quant(X, p, None, Xop, xs, sg, ws=ws)
    Y2 = torch.empty_like(Y1)
    rrs.rrs_gemm(Xop, xs, sg, layer.Wop, layer.w_scale, Y2, 1.0 / 4096)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    assert y_normalised_error(Y1.cpu().numpy(), ref) <= 1e-5


def test_deterministic_run_to_run():
    X_bits, W_bits, perm, _ = _gemm_case(300, 600, 1024)
    layer = rrs.RRSLinear(dev_bf16(W_bits), torch.from_numpy(perm).to(DEV))
    X = dev_bf16(X_bits)
    a = layer(X, out_dtype=torch.float32)
    b = layer(X, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_comm_world1_path_equals_single_gpu():
    """Column-parallel path with a 1-rank NCCL communicator (shard -> all-gather -> relayout)."""
    X_bits, W_bits, perm, ref = _gemm_case(130, 512, 1024)
    uid = rrs.rrs_comm_unique_id()
    comm = rrs.rrs_comm_init(0, 1, uid)
    try:
        p = torch.from_numpy(perm).to(DEV)
        single = rrs.RRSLinear(dev_bf16(W_bits), p)
        par = rrs.RRSLinear(dev_bf16(W_bits), p, comm=comm, world=1, rank=0)
        X = dev_bf16(X_bits)
        a = single(X, out_dtype=torch.float32)
        b = par(X, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    finally:
        rrs.rrs_comm_destroy(comm)


@pytest.mark.parametrize("K,T,i8", [(4096, 200, False), (14336, 70, False), (1024, 0, False), (2048, 150, True)])
def test_token_sharded_world1_equals_single_gpu(K, T, i8):
    """Token-sharded data parallel (RRS_TOKEN_SHARDED) with a 1-rank communicator: the two-pass
    prologue + ncclAllReduce(MAX) of chan_max + GEMM equals the single-GPU layer (fused prologue for 2^m)
    bit for bit; T = 0 still joins the collective."""
    X_bits = make_activations("mixed", T, K, 940, 941)
    W_bits = make_weights(264, K, 942)
    perm = _perm(make_activations("mixed", 64, K, 940, 943))
    uid = rrs.rrs_comm_unique_id()
    comm = rrs.rrs_comm_init(0, 1, uid)
    try:
        p = torch.from_numpy(perm).to(DEV)
        single = rrs.RRSLinear(dev_bf16(W_bits), p, i8=i8)
        dp = rrs.RRSLinear(dev_bf16(W_bits), p, comm=comm, world=1, rank=0, token_sharded=True, i8=i8)
        X = dev_bf16(X_bits)
        a = single(X, out_dtype=torch.float32)
        b = dp(X, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert b.shape == (T, 264) and torch.equal(a, b)
        if T:
            ref = oracle_layer(X_bits, W_bits, perm)
            assert y_normalised_error(b.cpu().numpy(), ref) <= 1e-5
    finally:
        rrs.rrs_comm_destroy(comm)


@pytest.mark.parametrize("T,out", [(2048, torch.bfloat16), (1100, torch.float32)])
def test_comm_slab_pipeline_equals_single_gpu(T, out):
    """Column-parallel path through NCCL (1-rank communicator) with T >= 1024: the GEMM runs in 256-row-aligned
    token slabs and each slab's all-gather + relayout runs on the side stream, overlapping the next slab's GEMM
    (SURVEY §8(e)).  Bitwise equal to the single-GPU layer (ragged last slab at T = 1100)."""
    X_bits, W_bits, perm, _ = _gemm_case(T, 512, 1024, "channel", seed=3)
    uid = rrs.rrs_comm_unique_id()
    comm = rrs.rrs_comm_init(0, 1, uid)
    try:
        p = torch.from_numpy(perm).to(DEV)
        single = rrs.RRSLinear(dev_bf16(W_bits), p)
        par = rrs.RRSLinear(dev_bf16(W_bits), p, comm=comm, world=1, rank=0)
        X = dev_bf16(X_bits)
        a = single(X, out_dtype=out)
        for _ in range(2):  # back-to-back calls reuse the shard / gather buffers and the side stream
            b = par(X, out_dtype=out)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    finally:
        rrs.rrs_comm_destroy(comm)


def test_perm_helper_matches_oracle():
    K = 4096
    Xc = make_activations("channel", 64, K, 11, 12)
    Xr = torch.empty((64, K), dtype=torch.float32, device=DEV)
    cm = torch.empty(K, dtype=torch.float32, device=DEV)
    rrs.rrs_debug_rotate(dev_bf16(Xc), Xr, cm)
    perm = torch.empty(K, dtype=torch.int32, device=DEV)
    rrs.rrs_perm_from_channel_max(cm, perm)
    torch.cuda.synchronize()
    assert np.array_equal(perm.cpu().numpy(), _perm(Xc))
    # ties: ascending index (R21)
    c = torch.tensor([5, 5, 7, 5, 0, 7] + [0] * 122, dtype=torch.float32, device=DEV)
    pp = torch.empty(128, dtype=torch.int32, device=DEV)
    rrs.rrs_perm_from_channel_max(c, pp)
    assert np.array_equal(pp.cpu().numpy(), o.perm_from_channel_max(c.cpu().numpy()))


def test_invalid_arguments_raise():
    X = torch.zeros((4, 256), dtype=torch.bfloat16, device=DEV)
    p = torch.arange(256, dtype=torch.int32, device=DEV)
    xs = torch.empty(4, device=DEV)
    sg = torch.empty(2, device=DEV)
    with pytest.raises(rrs.RRSError) as e:
        rrs.rrs_rotate_smooth_quant(X, p, None, None, xs, sg, chan_max=torch.empty(256, device=DEV), group=48)
    assert e.value.status == 1  # not a power of two
    with pytest.raises(rrs.RRSError) as e:
        rrs.rrs_rotate_smooth_quant(X, p, None, None, xs, sg, chan_max=torch.empty(256, device=DEV), group=2048)
    assert e.value.status == 1  # above 1024
    Xbad = torch.zeros((4, 96 * 3), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(rrs.RRSError) as e:
        rrs.rrs_rotate_smooth_quant(Xbad, p, None, None, xs, sg, chan_max=torch.empty(288, device=DEV))
    assert e.value.status == 2


# ------------------------------------------------------------------------------------- full size, sampled

def test_full_size_c3_up_sampled():
    """The bench.py headline at full size (configs[2] up_proj: 4096 x 4096 x 14336, bf16 Y through rrs_linear,
    the bench's launch configuration): the prologue is checked in full (oracle rotation of all 4096 tokens:
    every s_g, alpha_t and code); Y on 48 sampled token rows x 64 sampled output features (the oracle prepares
    only those weight rows), both against the same oracle arithmetic."""
    w = WORKLOADS["c3_llama3_8b_up"]
    X_bits, W_bits, Xc = make_layer(w, index=list(WORKLOADS).index("c3_llama3_8b_up"))
    perm = _perm(Xc[:256])
    p = torch.from_numpy(perm).to(DEV)
    g = _run_prologue(X_bits, perm)
    Xr = o.rotate(bf16_bits_to_f64(X_bits))
    s = o.group_scales(o.channel_max(Xr), perm, 128)
    q, a = o.smooth_quant(Xr, perm, s, 128)
    assert np.array_equal(g["s_group"].view(np.uint32), s.view(np.uint32))
    assert np.array_equal(g["alpha"].view(np.uint32), a.view(np.uint32))
    assert np.array_equal(g["Xq8"], q)
    layer = rrs.RRSLinear(dev_bf16(W_bits), p)
    Y = layer(dev_bf16(X_bits), out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    rows = rng.choice(w.T, size=48, replace=False)
    cols = np.sort(rng.choice(w.N, size=64, replace=False))
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits[cols]), perm)
    assert np.array_equal(layer.w_scale.cpu().numpy()[cols].view(np.uint32), beta.view(np.uint32))
    P = o.group_partials(q[rows], qw, 128)
    Yref = o.scale_accumulate(P, s, a[rows], beta, 1.0 / w.K)
    ref = dict(P=P, s_group=s, alpha=a[rows], beta=beta, out_scale=1.0 / w.K, Y=Yref)
    Ys = Y.float().cpu().numpy()[np.ix_(rows, cols)]
    assert bf16_ulp_error(Ys, Yref, ref) <= 1.0


def test_full_size_c3_down_sampled():
    """configs[2] down_proj at full size (4096 x 14336 x 4096, K = 28 * 512, spike-profile activations), bf16 Y
    through rrs_linear: every code of the prologue, Y on sampled rows x columns (as above)."""
    w = WORKLOADS["c3_llama3_8b_down"]
    X_bits, W_bits, Xc = make_layer(w, index=list(WORKLOADS).index("c3_llama3_8b_down"))
    perm = _perm(Xc[:256])
    p = torch.from_numpy(perm).to(DEV)
    g = _run_prologue(X_bits, perm)
    Xr = o.rotate(bf16_bits_to_f64(X_bits))
    s = o.group_scales(o.channel_max(Xr), perm, 128)
    q, a = o.smooth_quant(Xr, perm, s, 128)
    assert np.array_equal(g["s_group"].view(np.uint32), s.view(np.uint32))
    assert np.array_equal(g["alpha"].view(np.uint32), a.view(np.uint32))
    assert np.array_equal(g["Xq8"], q)
    layer = rrs.RRSLinear(dev_bf16(W_bits), p)
    Y = layer(dev_bf16(X_bits), out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    rng = np.random.default_rng(2)
    rows = rng.choice(w.T, size=48, replace=False)
    cols = np.sort(rng.choice(w.N, size=64, replace=False))
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits[cols]), perm)
    P = o.group_partials(q[rows], qw, 128)
    Yref = o.scale_accumulate(P, s, a[rows], beta, 1.0 / w.K)
    ref = dict(P=P, s_group=s, alpha=a[rows], beta=beta, out_scale=1.0 / w.K, Y=Yref)
    assert bf16_ulp_error(Y.float().cpu().numpy()[np.ix_(rows, cols)], Yref, ref) <= 1.0


def test_full_size_c2_sampled_rows():
    """BASELINE configs[1] at full size (2048 x 4096 x 4096), same launch configuration as bench.py.

    The prologue is checked in full (oracle rotation of all 2048 tokens); Y on 64 sampled token rows
    (the oracle's grouped GEMM restricted to those rows, exact same arithmetic)."""
    w = WORKLOADS["c2_llama2_7b_qo"]
    X_bits, W_bits, Xc = make_layer(w, index=1)
    perm = _perm(Xc[:256])
    X = dev_bf16(X_bits)
    p = torch.from_numpy(perm).to(DEV)
    g = _run_prologue(X_bits, perm)
    Xr = o.rotate(bf16_bits_to_f64(X_bits))
    c = o.channel_max(Xr)
    s = o.group_scales(c, perm, 128)
    q, a = o.smooth_quant(Xr, perm, s, 128)
    assert np.array_equal(g["s_group"].view(np.uint32), s.view(np.uint32))
    assert np.array_equal(g["alpha"].view(np.uint32), a.view(np.uint32))
    assert np.array_equal(g["Xq"], o.pack_int4(q))
    layer = rrs.RRSLinear(dev_bf16(W_bits), p)
    Y = layer(X, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = np.random.default_rng(0).choice(w.T, size=64, replace=False)
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits), perm)
    assert np.array_equal(layer.w_scale.cpu().numpy().view(np.uint32), beta.view(np.uint32))
    P = o.group_partials(q[rows], qw, 128)
    Yref = o.scale_accumulate(P, s, a[rows], beta, 1.0 / w.K)
    ref = dict(P=P, s_group=s, alpha=a[rows], beta=beta, out_scale=1.0 / w.K, Y=Yref)
    assert y_normalised_error(Y.cpu().numpy()[rows], ref) <= 1e-5
