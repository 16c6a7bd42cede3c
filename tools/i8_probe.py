"""int8 tensor-core gather (the default engine) vs the FP64 DMMA gather and the
reference goldens: accuracy (rel-linf) and forward window-stage time."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_10786_b200 as sgl  # noqa: E402
from paper_1809_10786_b200 import workloads  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def mk(B, pts, rho, q=16, i8=False, sigma=2):
    # default backend: int8 tensor-core gather; "tiled": the FP64 DMMA gather
    return sgl.plan(B, pts, rho=rho, q=q, sigma=sigma, profile=True, backend="auto" if i8 else "tiled")


ap = argparse.ArgumentParser()
ap.add_argument("--big", type=int, default=10_000_000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

gd = os.path.join(ROOT, "tests", "golden")
for name in ["ref_b12_q12.npz", "ref_b8_q16.npz", "ref_cfg1.npz", "ref_cfg3_sub600.npz", "ref_edges_b8_q16.npz",
             "ref_cfg5_sub400.npz", "ref_b4_q8.npz"]:
    g = np.load(os.path.join(gd, name))
    B, q, rho = int(g["B"]), int(g["q"]), float(g["rho"])
    sigma = int(g["sigma"]) if "sigma" in g else 2
    c = g["coeffs"] if g["coeffs"].ndim == 1 else g["coeffs"][0]
    fref = g["fwd"] if g["fwd"].ndim == 1 else g["fwd"][0]
    try:
        p8 = mk(B, g["points"], rho, q, True, sigma)
        p6 = mk(B, g["points"], rho, q, False, sigma)
        f8 = sgl.forward(p8, c)
        f6 = sgl.forward(p6, c)
        print(f"{name}: B={B} q={q} M={p8.m_points} i8 vs ref {rel(f8, fref):.2e}  fp64 vs ref {rel(f6, fref):.2e}  "
              f"i8 vs fp64 {rel(f8, f6):.2e}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name}: ERROR {e}", flush=True)

for cfg, M in [(3, 1_000_000), (3, a.big), (1, None), (2, None), (5, None)]:
    w = workloads.config(cfg, M=M)
    c = w.coeffs if w.coeffs.ndim == 1 else w.coeffs[0]
    out = {}
    for i8 in (False, True):
        t0 = time.time()
        p = mk(w.B, w.points, w.rho, 16, i8)
        tp = time.time() - t0
        f = sgl.forward(p, c)
        ms = []
        for _ in range(a.reps):
            f = sgl.forward(p, c)
            ms.append(p.stage_ms("forward")["window"])
        out[i8] = (f, min(ms), tp, p.stats)
        p.close()
    print(f"cfg{cfg} M={w.M}: window fp64 {out[False][1]:.3f} ms  i8 {out[True][1]:.3f} ms  "
          f"(x{out[False][1] / out[True][1]:.2f})  i8 vs fp64 rel-linf {rel(out[True][0], out[False][0]):.2e}  "
          f"plan {out[False][2]:.2f}/{out[True][2]:.2f} s", flush=True)
