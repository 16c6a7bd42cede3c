"""Numpy model of the int8 digit-split window gather (gather_i8.cu) on a
reference golden case: error of several digit / diagonal configurations
against the FP64 window sum (the oracle's grid and window tables).

    python tools/ozaki_sim.py [golden.npz ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import sgl_oracle as o  # noqa: E402

MAGIC = 1.5 * 2.0 ** 52


def digits_unsigned(x_fix, nd):
    x = x_fix.astype(np.int64)
    return np.stack([(x >> (8 * j)) & 255 for j in range(nd)]).astype(np.float64)


def digits_balanced(x_fix, nd):
    f = x_fix.astype(np.int64).copy()
    out = []
    for _ in range(nd):
        d = ((f + 128) & 255) - 128
        out.append(d)
        f = (f - d) >> 8
    assert np.all(f == 0)
    return np.stack(out).astype(np.float64)


def sim(grid, p, na, nb, dmin, abal=False, per_b=False):
    q = p.q
    N = np.array(grid.shape)
    offs = np.arange(2 * q + 1)
    c = [(N[j] / (2 * np.pi)) / np.sqrt(2 * np.pi * p.lam[j]) for j in range(3)]
    eA = int(np.ceil(np.log2(c[0] * c[2])))
    tA = 8 * na - 1          # A 2^sA < 2^tA
    sA = tA - eA
    gmax = max(np.abs(grid.real).max(), np.abs(grid.imag).max())
    ex = int(np.frexp(gmax)[1])
    tB = 8 * nb - 2          # |G| 2^sG < 2^tB
    sG = tB - ex
    M = p.m_points
    out = np.zeros(M, complex)
    ref = np.zeros(M, complex)
    for i in range(M):
        idx = [(p.base[j][i] - q + offs) % N[j] for j in range(3)]
        sub = grid[np.ix_(idx[0], idx[1], idx[2])]
        w0, w1, w2 = p.win[0][i], p.win[1][i], p.win[2][i]
        ref[i] = np.einsum("abc,a,b,c->", sub, w0, w1, w2)
        A = np.outer(w0, w2)                                # (a, c)
        Afix = np.rint(A * 2.0 ** sA)
        ad = digits_balanced(Afix, na) if abal else digits_unsigned(Afix, na)   # (na, a, c)
        res = 0j
        for part, gpart in ((1.0, sub.real), (1j, sub.imag)):
            Gfix = np.rint(gpart * 2.0 ** sG)
            bd = digits_balanced(Gfix, nb)                  # (nb, a, b, c)
            # D_pq[b] = sum_{a,c} a_p[a,c] b_q[a,b,c]   (exact in float64)
            D = np.einsum("pac,qabc->pqb", ad, bd, optimize=True)
            v = np.zeros(D.shape[2])
            for d in range(na + nb - 2, dmin - 1, -1):      # most significant first (kernel: least first)
                for pp in range(na):
                    qq = d - pp
                    if 0 <= qq < nb:
                        v = v + D[pp, qq] * 2.0 ** (8 * d)
            res += part * np.dot(w1, v) * 2.0 ** (-sA - sG)
        out[i] = res
    return out, ref


def main():
    names = sys.argv[1:] or ["ref_cfg5_sub400.npz", "ref_cfg1.npz"]
    for name in names:
        g = np.load(os.path.join(ROOT, "tests", "golden", name))
        B, q, rho = int(g["B"]), int(g["q"]), float(g["rho"])
        c = g["coeffs"] if g["coeffs"].ndim == 1 else g["coeffs"][0]
        fref = g["fwd"] if g["fwd"].ndim == 1 else g["fwd"][0]
        pts = g["points"][:200]
        p = o.oracle_plan(B, pts, q=q, rho=rho)
        grid = o.spectral_forward(p, o.basal_forward(p, c))
        gmax = np.abs(grid).max()
        print(f"{name}: B={B} M={p.m_points} max|G|={gmax:.3e} max|f|={np.abs(fref[:200]).max():.3e}")
        for na, nb, dmin, abal in [(6, 6, 5, False), (6, 6, 5, True), (6, 6, 4, False), (6, 6, 4, True), (6, 6, 6, True)]:
            out, ref = sim(grid, p, na, nb, dmin, abal)
            e = np.abs(out - ref).max() / np.abs(ref).max()
            print(f"  A {na} {'balanced' if abal else 'unsigned'} digits, B {nb} digits, keep p+q >= {dmin} "
                  f"({sum(1 for a in range(na) for b in range(nb) if a + b >= dmin)} pairs, "
                  f"{na + nb - 1 - dmin} diagonals): rel-linf {e:.2e}")


if __name__ == "__main__":
    main()
