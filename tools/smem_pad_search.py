"""Search the shared-memory padding of the FWHT transpose tile (fwht.cuh) for conflict-free 8-byte accesses.

pad(i) = i + sum_s c_s * (i >> s) is strictly increasing (hence injective) for any c_s >= 0.  For every
access pattern of a plan (pass-0 stores, middle-pass loads/stores, H28 loads) and every register index,
the 32 lanes of a warp access doubles; 8-byte accesses are served per half-warp, conflict-free iff the 16
lanes of each half hit 16 distinct 8-byte slots (pad mod 16).  Prints excess wavefronts per pattern.
"""
import itertools
import sys


def plan(K):
    pow2 = K & (K - 1) == 0
    A = 1 if pow2 else 28
    NP2 = K // A
    LOGN = NP2.bit_length() - 1
    B = 5
    E = 1 << B
    TP2 = K // E
    TH28 = 0 if pow2 else NP2  # one 28-vector per thread in the H28 pass
    HI = LOGN - (B - 3)
    return dict(K=K, pow2=pow2, NP2=NP2, LOGN=LOGN, B=B, E=E, TP2=TP2, TH28=TH28, HI=HI)


def p0_index(P, tp, j):
    per_chunk = P["NP2"] // P["E"]
    a, t = divmod(tp, per_chunk)
    return a * P["NP2"] + ((j >> 3) << P["HI"]) + (t << 3) + (j & 7)


def p2_index(P, b, r, tp, u, k):
    g = tp + P["TP2"] * u
    return (g & ((1 << b) - 1)) | (k << b) | ((g >> b) << (b + r))


def layouts(P):
    out = [("p0", lambda tp, j: p0_index(P, tp, j), P["E"], P["TP2"])]
    b = 3
    while b < P["HI"]:
        r = min(P["B"], P["HI"] - b)
        out.append((f"mid{b}", (lambda b, r: lambda tp, j: p2_index(P, b, r, tp, j >> r, j & ((1 << r) - 1)))(b, r),
                    P["E"], P["TP2"]))
        b += r
    if not P["pow2"]:
        out.append(("h28", lambda tp, j: j * P["NP2"] + tp, 28, P["TH28"]))
    return out


def excess(P, coef, verbose=False):
    tot = 0
    for name, f, n, nthreads in layouts(P):
        ex = 0
        for j in range(n):
            for w0 in range(0, min(nthreads, 128), 32):
                for h in (0, 16):
                    slots = {}
                    for t in range(w0 + h, w0 + h + 16):
                        if t >= nthreads:
                            continue
                        i = f(t, j)
                        p = i + sum(c * (i >> s) for s, c in coef)
                        slots[p % 16] = slots.get(p % 16, 0) + 1
                    ex += max(slots.values()) - 1 if slots else 0
        if verbose:
            print(f"   {name}: excess {ex}")
        tot += ex
    return tot


def search(K):
    P = plan(K)
    best = None
    shifts = range(4, 12)
    for c4 in (1,):
        for (s1, c1), (s2, c2) in itertools.product([(s, c) for s in shifts for c in (0, 4, 8)], repeat=2):
            if s1 >= s2:
                continue
            coef = [(4, c4)] + [(s1, c1), (s2, c2)]
            e = excess(P, coef)
            if best is None or e < best[0]:
                best = (e, coef)
            if e == 0:
                return best
    return best


if __name__ == "__main__":
    for K in [int(x) for x in sys.argv[1:]] or [256, 1024, 2048, 4096, 8192, 16384, 7168, 14336]:
        P = plan(K)
        cur = [(4, 1), (9, 8)]
        print(K, "current pad excess", excess(P, cur))
        e, coef = search(K)
        print(K, "best", e, coef)
        excess(P, coef, verbose=True)
