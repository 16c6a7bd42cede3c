"""Config-3 forward with the int8 gather (the default engine) for ncu: plan + reps forwards."""
import os, sys, argparse
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=10_000_000)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--config", type=int, default=3)
a = ap.parse_args()
import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import workloads
w = workloads.config(a.config, M=a.m)
p = sgl.plan(w.B, w.points, rho=w.rho)
c = w.coeffs if w.coeffs.ndim == 1 else w.coeffs[0]
for _ in range(a.reps):
    f = sgl.forward(p, c)
print("ok", p.stats, float(np.abs(f).max()))
