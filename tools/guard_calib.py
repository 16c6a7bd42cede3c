"""Calibration of the int8 accuracy guard (csrc/guard.cu): per input family the
measured int8-vs-FP64 rel-linf and the guard's estimate (kappa = 1).  The
estimate must bound the measurement (ratio est/err >= 1) on every family,
and stay below the 1e-11 switch on the BASELINE configurations."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_10786_b200 as sgl  # noqa: E402
from paper_1809_10786_b200 import _native, indexing, workloads  # noqa: E402

NG = _native.FLAG_NO_GUARD


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def row(name, e, est):
    print(f"{name:48s} err {e:9.2e}  est {est:9.2e}  est/err {est / max(e, 1e-300):9.2e}", flush=True)


def fwd(name, p8, p64, c):
    f8, f64 = sgl.forward(p8, c), sgl.forward(p64, c)
    row("fwd " + name, rel(f8, f64), p8.guard["est_fwd"])


def adj(name, p8, p64, v):
    a8, a64 = sgl.adjoint(p8, v), sgl.adjoint(p64, v)
    row("adj " + name, rel(a8, a64), p8.guard["est_adj"])


rng = np.random.default_rng(0)
# BASELINE configurations (false-positive check)
for cfg, M in [(1, None), (2, None), (3, 1_000_000), (5, 200_000), (4, 2_000_000)]:
    w = workloads.config(cfg, M=M)
    p8 = sgl.plan(w.B, w.points, rho=w.rho, backend="i8", flags=NG)
    p64 = sgl.plan(w.B, w.points, rho=w.rho, backend="tiled")
    c = w.coeffs if w.coeffs.ndim == 1 else w.coeffs[0]
    if cfg != 4:
        fwd(f"cfg{cfg} M={w.M}", p8, p64, c)
    v = w.values if w.values is not None else rng.uniform(-1, 1, w.M) + 0j
    adj(f"cfg{cfg} M={w.M}", p8, p64, v)
    p8.close()
    p64.close()

# SGL corners
for B in (8, 16, 32):
    pts = sgl.gen_points_ball(20000, 2.0 + B / 8, rng)
    p8, p64 = sgl.plan(B, pts, backend="i8", flags=NG), sgl.plan(B, pts, backend="tiled")
    for n, l, m in [(B, B - 1, B - 1), (B, 0, 0), (1, 0, 0), (B, B - 1, 0)]:
        c = np.zeros(p8.count, complex)
        c[indexing.nlm_to_mu(n, l, m)] = 1.0
        fwd(f"B={B} single ({n},{l},{m})", p8, p64, c)
    nlm = indexing.mu_to_nlm_array(B)
    c = np.where(np.abs(nlm[:, 2]) == B - 1, sgl.gen_coeffs(B, rng), 0)
    fwd(f"B={B} edge |m|=B-1", p8, p64, c)
    for kind in ("uniform", "sparse5", "smooth"):
        if kind == "uniform":
            v = rng.uniform(-1, 1, 20000) + 1j * rng.uniform(-1, 1, 20000)
        elif kind == "sparse5":
            v = np.zeros(20000, complex)
            v[rng.choice(20000, 5)] = 1.0
        else:
            v = np.exp(-pts[:, 0] ** 2).astype(complex)
        adj(f"B={B} values {kind}", p8, p64, v)

# raw NFFT families
for n in [(32, 32, 32), (64, 64, 32)]:
    nodes = rng.uniform(0, 2 * np.pi, (50000, 3))
    p8 = sgl.nfft_plan(3, n, 2, 16, nodes, backend="i8")
    p64 = sgl.nfft_plan(3, n, 2, 16, nodes)
    for kind in ("white", "deconv_edge", "corner", "lowpass"):
        f = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        if kind == "deconv_edge":
            for ax, d in enumerate(p64.deconv):
                f = f * np.expand_dims(d, tuple(a for a in range(3) if a != ax))
        elif kind == "corner":
            f = np.zeros(n, complex)
            f[0, 0, 0] = 1
        elif kind == "lowpass":
            k = np.meshgrid(*[np.arange(x) - x // 2 for x in n], indexing="ij")
            f = f * np.exp(-(k[0] ** 2 + k[1] ** 2 + k[2] ** 2) / 20.0)
        o8, o64 = sgl.nfft_execute(p8, f), sgl.nfft_execute(p64, f)
        g = p8.guard
        row(f"nfft {n} {kind} (fallbacks {g['fwd_fallbacks']})", rel(o8, o64), g["est_fwd"])
