"""Decode regime (BASELINE configs[3]: 1-64 tokens x K = 8192 x N = 8192) through the packed-W path
(rrs.h RRS_W_PACKED4, csrc/decode.cu) against the CPU oracle.

Bar: packed W bytes bit-exact (the decode4 layout is written out here from the header's text, from
the oracle's integer codes); Y f32 within normalised error 1e-5, Y bf16 within 1 bf16 ulp (+ the FP32
allowance), at ragged T / N, both group sizes the decode kernel takes, and at the full configs[3] size.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2409_20361_b200 as rrs  # noqa: E402
from oracle import rrs_oracle as o  # noqa: E402
from rrs_synth import WORKLOADS, bf16_bits_to_f64, make_activations, make_layer, make_weights  # noqa: E402

from _parity import bf16_ulp_error, dev_bf16, encode_operand, oracle_layer, y_normalised_error  # noqa: E402

DEV = "cuda"


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def pack_decode4_rows(q: np.ndarray) -> np.ndarray:
    """Per row, per 32-code chunk j0: byte b (0..15) = (q[j0+b] & 0xF) << 4 | (q[j0+16+b] & 0xF) (rrs.h)."""
    q = np.asarray(q, dtype=np.int16)
    R, K = q.shape
    c = q.reshape(R, K // 32, 2, 16)
    return (((c[:, :, 0, :] & 0xF) << 4) | (c[:, :, 1, :] & 0xF)).astype(np.uint8).reshape(R, K // 2)


def _slot_perm():
    """Byte offset inside a tile row of chunk c is 16 (c ^ ((r >> 1) & 3)) (rrs.h RRS_W_PACKED4)."""
    r = np.arange(256)[:, None]
    c = np.arange(4)[None, :]
    return c ^ ((r >> 1) & 3)  # [256][4] slot of chunk c in row r


def tile_decode4(rows: np.ndarray, K: int) -> np.ndarray:
    """Row-major chunk bytes [N][K/2] -> the tiled layout: ceil(N/256) x K/128 tiles of [256 rows][4 slots][16 B]."""
    N = rows.shape[0]
    Np = (N + 255) // 256 * 256
    r = np.zeros((Np, K // 2), np.uint8)
    r[:N] = rows
    ch = r.reshape(Np // 256, 256, K // 128, 4, 16)              # [rb][row][kb][chunk][16]
    out = np.zeros((Np // 256, K // 128, 256, 4, 16), np.uint8)  # [rb][kb][row][slot][16]
    slot = _slot_perm()
    for row in range(256):
        for c in range(4):
            out[:, :, row, slot[row, c], :] = ch[:, row, :, c, :]
    return out.reshape(Np, K // 2)


def untile_decode4(tiled: np.ndarray, N: int, K: int) -> np.ndarray:
    Np = tiled.shape[0]
    t = tiled.reshape(Np // 256, K // 128, 256, 4, 16)
    rows = np.zeros((Np // 256, 256, K // 128, 4, 16), np.uint8)
    slot = _slot_perm()
    for row in range(256):
        for c in range(4):
            rows[:, row, :, c, :] = t[:, :, row, slot[row, c], :]
    return rows.reshape(Np, K // 2)[:N]


def pack_decode4(q: np.ndarray) -> np.ndarray:
    return tile_decode4(pack_decode4_rows(q), q.shape[1])


def _case(T, N, K, profile, seed=0, group=128):
    X_bits = make_activations(profile, T, K, 2100 + seed, 2101 + seed)
    W_bits = make_weights(N, K, 2102 + seed)
    perm = o.calibrate_perm(bf16_bits_to_f64(make_activations(profile, 64, K, 2100 + seed, 2103 + seed))).astype(np.int32)
    ref = oracle_layer(X_bits, W_bits, perm, group=group)
    return X_bits, W_bits, perm, ref


def test_pack_decode4_layout_by_hand():
    """The test's own packer against hand-worked bytes (the header's formula): codes 0..15 of a chunk -> high
    nibbles, 16..31 -> low nibbles, two's complement; tile placement and the slot swizzle."""
    q = np.zeros((1, 32), np.int8)
    q[0, 0], q[0, 16] = -1, 7      # byte 0 = 0xF << 4 | 7 = 0xF7
    q[0, 15], q[0, 31] = 3, -8     # byte 15 = 0x3 << 4 | 0x8 = 0x38
    b = pack_decode4_rows(q)[0]
    assert b[0] == 0xF7 and b[15] == 0x38 and not b[1:15].any()
    # row 3 (slot swizzle (3 >> 1) & 3 = 1), K-block 1, chunk 2 of row-block 1: q[259][128 + 64] = 5
    N, K = 300, 256
    q = np.zeros((N, K), np.int8)
    q[259, 192] = 5
    t = pack_decode4(q)
    assert t.shape == (512, 128)
    flat = t.reshape(-1)
    off = (1 * (K // 128) + 1) * 16384 + 3 * 64 + 16 * (2 ^ 1)
    assert flat[off] == 0x50 and np.count_nonzero(flat) == 1
    assert np.array_equal(untile_decode4(t, N, K), pack_decode4_rows(q))


@pytest.mark.parametrize("N,K", [(300, 1024), (256, 8192)])
def test_prepare_weights_packed4_bitexact(N, K):
    W_bits = make_weights(N, K, 2110)
    perm = o.calibrate_perm(bf16_bits_to_f64(make_activations("mixed", 64, K, 5, 6))).astype(np.int32)
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits), perm)
    Wp4 = torch.full(((N + 255) // 256 * 256, K // 2), 0xAB, dtype=torch.uint8, device=DEV)
    ws = torch.empty(N, dtype=torch.float32, device=DEV)
    rrs.rrs_prepare_weights(dev_bf16(W_bits), _dev(perm), None, Wp4, ws, packed4=True)
    torch.cuda.synchronize()
    assert np.array_equal(Wp4.cpu().numpy(), pack_decode4(qw))
    assert np.array_equal(ws.cpu().numpy().view(np.uint32), beta.view(np.uint32))


@pytest.mark.parametrize("T,N,K,group,profile", [(1, 512, 1024, 128, "mixed"), (5, 300, 2048, 128, "channel"),
                                                 (16, 264, 1024, 256, "spike"), (17, 520, 4096, 128, "mixed"),
                                                 (33, 256, 1024, 512, "mixed"), (64, 776, 8192, 128, "mixed"),
                                                 (64, 256, 128, 128, "tiny")])
def test_decode_gemm_packed4(T, N, K, group, profile):
    """rrs_gemm(RRS_W_PACKED4) on the oracle's codes: int8 X [T][K], decode4-packed W; Y f32 and bf16."""
    X_bits, W_bits, perm, ref = _case(T, N, K, profile, seed=T, group=group)
    Xq8 = _dev(encode_operand(ref["q"], True))
    Wp4 = _dev(pack_decode4(ref["qw"]))
    xs, sg, ws = (torch.from_numpy(ref[k]).to(DEV) for k in ("alpha", "s_group", "beta"))
    ldy = (N + 7) // 8 * 8
    Yf = torch.full((T, ldy), float("nan"), dtype=torch.float32, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wp4, ws, Yf[:, :N], 1.0 / K, group=group, packed4=True)
    Yb = torch.full((T, ldy), float("nan"), dtype=torch.bfloat16, device=DEV)
    rrs.rrs_gemm(Xq8, xs, sg, Wp4, ws, Yb[:, :N], 1.0 / K, group=group, packed4=True)
    torch.cuda.synchronize()
    Yf_np = Yf.cpu().numpy()
    assert np.isnan(Yf_np[:, N:]).all()
    assert y_normalised_error(Yf_np[:, :N], ref) <= 1e-5
    assert bf16_ulp_error(Yb[:, :N].float().cpu().numpy(), ref["Y"], ref) <= 1.0
    assert torch.equal(Yb[:, :N], Yf[:, :N].to(torch.bfloat16))


def test_decode_gemm_deterministic():
    T, N, K = 64, 1024, 8192
    X_bits, W_bits, perm, ref = _case(T, N, K, "mixed", seed=77)
    Xq8 = _dev(encode_operand(ref["q"], True))
    Wp4 = _dev(pack_decode4(ref["qw"]))
    xs, sg, ws = (torch.from_numpy(ref[k]).to(DEV) for k in ("alpha", "s_group", "beta"))
    Ys = []
    for _ in range(3):
        Y = torch.empty((T, N), dtype=torch.float32, device=DEV)
        rrs.rrs_gemm(Xq8, xs, sg, Wp4, ws, Y, 1.0 / K, packed4=True)
        Ys.append(Y)
    torch.cuda.synchronize()
    assert torch.equal(Ys[0], Ys[1]) and torch.equal(Ys[0], Ys[2])


@pytest.mark.parametrize("T", [1, 7, 64])
def test_rrs_linear_decode_layer(T):
    """RRSLinear(decode=True): prologue (int8 codes) + the packed-W GEMM, against the oracle layer."""
    X_bits, W_bits, perm, ref = _case(T, 1000, 8192, "mixed", seed=100 + T)
    layer = rrs.RRSLinear(dev_bf16(W_bits), _dev(perm), decode=True)
    assert layer.Wp4 is not None
    Y = layer(dev_bf16(X_bits), out_dtype=torch.float32)
    Yb = layer(dev_bf16(X_bits), out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert y_normalised_error(Y.cpu().numpy(), ref) <= 1e-5
    assert bf16_ulp_error(Yb.float().cpu().numpy(), ref["Y"], ref) <= 1.0


@pytest.mark.parametrize("wl", ["c4_decode_t64", "c4_decode_t1"])
def test_full_size_c4_decode(wl):
    """configs[3] at full size (T x 8192 x 8192) in bench.py's launch configuration: every code of the
    prologue is implied by Y on 96 sampled output features (the oracle prepares only those W rows)."""
    w = WORKLOADS[wl]
    X_bits, W_bits, Xc = make_layer(w, index=list(WORKLOADS).index(wl))
    perm = o.calibrate_perm(bf16_bits_to_f64(Xc)).astype(np.int32)
    layer = rrs.RRSLinear(dev_bf16(W_bits), _dev(perm), decode=True)
    Y = layer(dev_bf16(X_bits), out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    cols = np.sort(np.random.default_rng(4).choice(w.N, size=96, replace=False))
    Xr = o.rotate(bf16_bits_to_f64(X_bits))
    s = o.group_scales(o.channel_max(Xr), perm, 128)
    q, a = o.smooth_quant(Xr, perm, s, 128)
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits[cols]), perm)
    assert np.array_equal(untile_decode4(layer.Wp4.cpu().numpy(), w.N, w.K)[cols], pack_decode4_rows(qw))
    P = o.group_partials(q, qw, 128)
    Yref = o.scale_accumulate(P, s, a, beta, 1.0 / w.K)
    ref = dict(P=P, s_group=s, alpha=a, beta=beta, out_scale=1.0 / w.K, Y=Yref)
    assert bf16_ulp_error(Y.float().cpu().numpy()[:, cols], Yref, ref) <= 1.0


def test_decode_refuses_large_T_and_small_groups():
    K, N = 1024, 256
    Xq8 = torch.zeros((65, K), dtype=torch.uint8, device=DEV)
    Wp4 = torch.zeros((N, K // 2), dtype=torch.uint8, device=DEV)
    one = torch.ones(65, device=DEV)
    with pytest.raises(rrs.RRSError) as e:
        rrs.rrs_gemm(Xq8, one, torch.ones(K // 128, device=DEV), Wp4, torch.ones(N, device=DEV),
                     torch.empty((65, N), device=DEV), 1.0 / K, packed4=True)
    assert e.value.status == 2
    with pytest.raises(rrs.RRSError) as e:
        rrs.rrs_gemm(Xq8[:8], one[:8], torch.ones(K // 64, device=DEV), Wp4, torch.ones(N, device=DEV),
                     torch.empty((8, N), device=DEV), 1.0 / K, group=64, packed4=True)
    assert e.value.status == 2
