"""Where the int8 window kernels' MMA warps wait (SGL_FLAG_I8_PROF clock64
counters, printed to stderr by the library) at a BASELINE config."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import _native, workloads
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--m", type=int, default=None)
a = ap.parse_args()
w = workloads.config(a.config, M=a.m)
p = sgl.plan(w.B, w.points, rho=w.rho, flags=_native.FLAG_I8_PROF)
c = w.coeffs if w.coeffs.ndim == 1 else w.coeffs[0]
for _ in range(2):
    sgl.forward(p, c)
    if w.values is not None:
        sgl.adjoint(p, w.values)
