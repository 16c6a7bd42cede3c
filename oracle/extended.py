"""Extended-precision direct sums -- TEST INFRASTRUCTURE ONLY.

The truth against which the FP64 paths are judged where FP64 itself is not
enough (BASELINE config 4: B = 128, rho = 22, adjoint entries spanning
1 .. 1e95).  It restates the reference's direct adjoint
`evaluate_direct_adjoint` (transform.py:120-139) -- the "ground-truth oracle"
of the reference's own docstring (transform.py:1-4) -- with every recurrence,
normalisation and accumulation in numpy longdouble (x87 80-bit: 64-bit
mantissa, 11 bits more than FP64; the reference uses the same type for its
own `precise=True` mode, recurrences.py:13-16).  The inputs are the FP64
points and values as given; only the arithmetic is extended.

* radial family f_k(r) = N(k+l+1, l) L_k^{(l+1/2)}(r^2) r^l by the normalised
  three-term recurrence of `radial_recurrence` (recurrences.py:85-106);
* P_{lm}(cos theta) by the degree recurrence from the seeds of
  `legendre_seeds` (special.py:66-90; recurrences.py:60-82), m >= 0;
* Q(l, m) = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!) (special.py:133-146), negated
  for odd negative m (`_sph_norm_signed`, transform.py:84-92);
* c_mu = sum_i v_i conj(H_mu(x_i)) with mu = n(n-1)(2n-1)/6 + l(l+1) + m
  (transform.py:120-139, indexing.py:29-38).

Log-gamma values are sums of logs of exact integers / half-integers in
longdouble (no FP64 gammaln).  `mp_direct_adjoint_entries` recomputes chosen
entries with mpmath at 50 digits to pin this module itself.

Only `tests/` and `tests/golden/` scripts import it; never the product.
"""
from __future__ import annotations

import numpy as np

LD = np.longdouble
CLD = np.clongdouble
PI_LD = LD(4) * np.arctan(LD(1))


def _lgamma_half(k: int) -> LD:
    """log Gamma(k + 1/2) for integer k >= 1, exactly summed in longdouble."""
    v = np.log(np.sqrt(PI_LD))   # Gamma(1/2) = sqrt(pi)
    for j in range(k):
        v += np.log(LD(j) + LD(0.5))
    return v


def _lfact(k: int) -> LD:
    v = LD(0)
    for j in range(2, k + 1):
        v += np.log(LD(j))
    return v


def radial_table_ld(l: int, n: int, r: np.ndarray) -> np.ndarray:
    """(n, len(r)) f_0..f_{n-1} of `radial_recurrence(l)` (recurrences.py:85-106)."""
    r = np.asarray(r, dtype=LD)
    a = LD(l) + LD(0.5)
    c0 = np.exp(LD(0.5) * (np.log(LD(2)) - _lgamma_half(l + 1)))   # Gamma(l + 3/2)
    out = np.empty((n, r.size), dtype=LD)
    rl = r ** l
    r2 = r * r
    if n > 0:
        out[0] = c0 * rl
    if n > 1:
        out[1] = c0 / np.sqrt(LD(1) + a) * (LD(1) + a - r2) * rl
    for k in range(2, n):
        kk = k - 1
        alpha = (LD(2 * kk + 1) + a - r2) / LD(kk + 1) * np.sqrt(LD(kk + 1) / (LD(kk + 1) + a))
        beta = -np.sqrt(LD(kk) * (LD(kk) + a) / (LD(kk + 1) * (LD(kk + 1) + a)))
        out[k] = alpha * out[k - 1] + beta * out[k - 2]
    return out


def legendre_table_ld(m: int, n: int, x: np.ndarray) -> np.ndarray:
    """(n, len(x)) P_{m+k, m}(x), m >= 0 (special.py:66-90, recurrences.py:60-82)."""
    x = np.asarray(x, dtype=LD)
    # (2m-1)!! = (2m)! / (2^m m!)
    log_c = _lfact(2 * m) - LD(m) * np.log(LD(2)) - _lfact(m) if m > 0 else LD(0)
    sign = LD(-1) if m % 2 else LD(1)
    s2 = np.clip(LD(1) - x * x, LD(0), None)
    out = np.empty((n, x.size), dtype=LD)
    f0 = sign * np.exp(log_c) * s2 ** (LD(m) / LD(2))
    if n > 0:
        out[0] = f0
    if n > 1:
        out[1] = LD(2 * m + 1) * x * f0
    for k in range(2, n):
        l = m + k - 1
        out[k] = (LD(2 * l + 1) * x * out[k - 1] - LD(l + m) * out[k - 2]) / LD(l + 1 - m)
    return out


def sph_norm_ld(l: int, m: int) -> LD:
    return np.exp(LD(0.5) * (np.log(LD(2 * l + 1) / (LD(4) * PI_LD)) + _lfact(l - m) - _lfact(l + m)))


def direct_adjoint_ld(values: np.ndarray, B: int, points: np.ndarray, cos_fp64: bool = False) -> np.ndarray:
    """c_mu = sum_i v_i conj(H_mu(x_i)) in longdouble (transform.py:120-139).
    Returns clongdouble (count,).  ``cos_fp64``: take cos(theta) rounded to
    FP64 first, as the reference does (transform.py:127); near the poles
    (theta ~ 1e-9) that rounding alone changes P_lm(cos theta) for m > 0 at
    the 1e-10 level, so the pin against the reference's direct sums uses it,
    while the truth keeps the extended cos."""
    points = np.atleast_2d(np.asarray(points, dtype=float))
    v = np.asarray(values, dtype=complex).astype(CLD)
    r = points[:, 0].astype(LD)
    ct = np.cos(points[:, 1]).astype(LD) if cos_fp64 else np.cos(points[:, 1].astype(LD))
    phi = points[:, 2].astype(LD)
    M = points.shape[0]
    gt = np.zeros((B * B, M), dtype=CLD)
    for am in range(B):
        leg = legendre_table_ld(am, B - am, ct)               # rows l = am .. B-1
        q = np.array([sph_norm_ld(l, am) for l in range(am, B)], dtype=LD)
        ql = q[:, None] * leg
        for m in ((am, -am) if am else (0,)):
            # Q(l,-m) P_{l,-m} = (-1)^m Q(l,m) P_{lm} (transform.py:84-92)
            sgn = LD(-1) if (m < 0 and am % 2) else LD(1)
            ph = np.cos(LD(m) * phi) - 1j * np.sin(LD(m) * phi).astype(CLD)   # exp(-i m phi)
            rows = np.arange(am, B) * np.arange(am + 1, B + 1) + m
            gt[rows] = (sgn * ql).astype(CLD) * (v * ph)[None, :]
    out = np.empty(B * (B + 1) * (2 * B + 1) // 6, dtype=CLD)
    for l in range(B):
        rad = radial_table_ld(l, B - l, r).astype(CLD)          # n = l+1 .. B
        blk = gt[l * l:(l + 1) * (l + 1)] @ rad.T                # (2l+1, B-l)
        n = np.arange(l + 1, B + 1)
        for mm in range(-l, l + 1):
            mu = n * (n - 1) * (2 * n - 1) // 6 + l * (l + 1) + mm
            out[mu] = blk[mm + l]
    return out


def mp_direct_adjoint_entries(values, B, points, mus, dps=50):
    """Selected entries c_mu at `dps` decimal digits (mpmath), from the
    closed forms of the basis (special.py:1-16, 147-165): N(n,l) from Gamma
    functions, L_k^{(l+1/2)}(r^2) and P_l^m by mpmath, Condon-Shortley phase."""
    import mpmath as mp
    mp.mp.dps = dps
    out = []
    pts = np.atleast_2d(points)
    for mu in mus:
        mu = int(mu)
        n = 1
        while (n + 1) * n * (2 * n + 1) // 6 <= mu:
            n += 1
        rem = mu - n * (n - 1) * (2 * n - 1) // 6
        l = int(np.floor(np.sqrt(rem)))
        while l * l > rem:
            l -= 1
        while (l + 1) ** 2 <= rem:
            l += 1
        m = rem - l * (l + 1)
        am = abs(m)
        N = mp.sqrt(2 * mp.factorial(n - l - 1) / mp.gamma(n + mp.mpf(1) / 2))
        Q = mp.sqrt(mp.mpf(2 * l + 1) / (4 * mp.pi) * mp.factorial(l - am) / mp.factorial(l + am))
        acc = mp.mpc(0)
        for (r, th, ph), val in zip(pts, values):
            r, th, ph = mp.mpf(float(r)), mp.mpf(float(th)), mp.mpf(float(ph))
            R = N * mp.laguerre(n - l - 1, l + mp.mpf(1) / 2, r * r) * r ** l
            P = mp.legenp(l, am, mp.cos(th), type=2)   # includes (-1)^m (Condon-Shortley)
            Y = Q * P
            if m < 0 and am % 2:
                Y = -Y
            H = R * Y * mp.expj(m * ph)
            acc += mp.mpc(complex(val)) * mp.conj(H)
        out.append(complex(acc))
    return np.array(out)
