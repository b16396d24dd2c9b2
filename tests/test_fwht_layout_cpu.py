"""The FWHT kernels (csrc/fwht.cuh) address shared memory as base(thread) + constant(register): that is exact only if, in
every pass layout of every plan, the tile index splits into disjoint bit fields -- the row / thread part
reg_index(tp, 0) and the register part reg_index(0, j) -- because then every shift of the padding function swz
distributes over the sum.  This checks the property, and swz additivity, for every K the library builds (B = 5 and
B = 6 plans), written out from the header's index definitions."""
import pytest


def plan(K, B):
    pow2 = K & (K - 1) == 0
    A = 1 if pow2 else 28
    NP2 = K // A
    LOGN = NP2.bit_length() - 1
    E = 1 << B
    TP2 = K // E
    HI = LOGN - (B - 3)
    R = max(1, (128 if B == 5 else 64) // TP2) if pow2 else 1
    if pow2:
        pad = [(4, 1), (7 if B == 5 else 8, 4)]
    else:
        pad = [(4, 1)] + ([(6, 4), (8, 4)] if NP2 <= 256 else [])
    return dict(K=K, pow2=pow2, NP2=NP2, LOGN=LOGN, B=B, E=E, TP2=TP2, TH28=0 if pow2 else NP2, HI=HI, R=R, pad=pad)


def p0_index(P, tp, j):
    per_chunk = P["NP2"] // P["E"]
    a, t = divmod(tp, per_chunk)
    return a * P["NP2"] + ((j >> 3) << P["HI"]) + (t << 3) + (j & 7)


def p2_index(P, b, r, tp, u, k):
    g = tp + P["TP2"] * u
    return (g & ((1 << b) - 1)) | (k << b) | ((g >> b) << (b + r))


def layouts(P):
    """(index function, registers, threads, separable) per pass layout; `separable` = the kernel uses base + offset."""
    out = [(lambda tp, j: p0_index(P, tp, j), P["E"], P["TP2"], True)]
    b = 3
    while b < P["HI"]:
        r = min(P["B"], P["HI"] - b)
        out.append(((lambda b, r: lambda tp, j: p2_index(P, b, r, tp, j >> r, j & ((1 << r) - 1)))(b, r), P["E"],
                    P["TP2"], P["pow2"]))
        b += r
    if not P["pow2"]:
        out.append((lambda tp, j: j * P["NP2"] + tp, 28, P["TH28"], True))
    return out


def swz(P, i):
    return i + sum(c * (i >> s) for s, c in P["pad"])


CASES = [(K, 5) for K in (128, 256, 512, 1024, 2048, 4096, 8192, 16384, 7168, 14336)] + \
        [(K, 6) for K in (4096, 8192, 16384)]


@pytest.mark.parametrize("K,B", CASES)
def test_layout_fields_disjoint_and_swz_additive(K, B):
    P = plan(K, B)
    for f, n, nthreads, sep in layouts(P):
        if not sep:
            continue
        for rr in range(P["R"]):
            for tp in range(nthreads):
                base = rr * K + f(tp, 0)
                for j in range(n):
                    reg = f(0, j)
                    full = rr * K + f(tp, j)
                    assert base & reg == 0 and base + reg == full, (K, B, rr, tp, j)
                    assert swz(P, base) + swz(P, reg) == swz(P, full)
                    assert (full + (full >> 5)) == (base + (base >> 5)) + (reg + (reg >> 5))
