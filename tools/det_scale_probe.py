"""Adjoint of the int8 scatter vs the FP64 scatter over the FP64 range of
input scales, with and without SGL_FLAG_DETERMINISTIC."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, paper_1809_10786_b200 as sgl
rng = np.random.default_rng(5)
pts = sgl.gen_points_ball(4000, 4.0, rng)
v0 = (rng.standard_normal(4000) + 1j * rng.standard_normal(4000))
p64 = sgl.plan(16, pts, backend="tiled")
for det in (False, True):
    p = sgl.plan(16, pts, backend="i8", deterministic=det)
    for s in (1e-300, 1e-290, 1e-280, 1e-250, 1e-200, 1.0, 1e300):
        v = v0 * s
        a, r = sgl.adjoint(p, v), sgl.adjoint(p64, v)
        print(det, s, float(np.max(np.abs(a - r)) / np.max(np.abs(r))), p.guard)

# forward (int8 gather) over the same range of coefficient scales
c0 = sgl.gen_coeffs(16, rng)
p8 = sgl.plan(16, pts)
for s in (1e-300, 1e-290, 1e-250, 1.0, 1e250, 1e300):
    f8, f64 = sgl.forward(p8, c0 * s), sgl.forward(p64, c0 * s)
    ok = np.isfinite(f64).all()
    print("fwd", s, float(np.max(np.abs(f8 - f64)) / np.max(np.abs(f64))) if ok else "ref not finite", p8.guard)
