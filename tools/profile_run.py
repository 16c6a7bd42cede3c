"""Short device run for ncu / compute-sanitizer: config-3 shape (B=64, ball 16)
with a reduced node count; plan + 2 x (forward + adjoint) on cuda:0."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10786_b200 as sgl  # noqa: E402
from paper_1809_10786_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--m", type=int, default=2_000_000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--backend", default="auto")
ap.add_argument("--profile", action="store_true", help="SGL_FLAG_I8_PROF: int8 kernel wait counters on stderr")
a = ap.parse_args()
w = workloads.config(a.config, M=a.m)
p = sgl.plan(w.B, w.points, rho=w.rho, backend=a.backend,
             flags=(1 << 12) if a.profile else 0)   # SGL_FLAG_I8_PROF
c = w.coeffs if w.coeffs.ndim == 1 else w.coeffs[0]
for _ in range(a.reps):
    f = sgl.forward(p, c)
    g = sgl.adjoint(p, w.values)
print("ok", p.stats, float(np.abs(f).max()), float(np.abs(g).max()))
