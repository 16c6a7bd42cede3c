"""int8 tensor-core scatter (backend="i8") vs the FP64 scatter (backend="tiled") and the
reference goldens: accuracy (rel-linf) and adjoint window-stage time."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_10786_b200 as sgl  # noqa: E402
from paper_1809_10786_b200 import workloads  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def mk(B, pts, rho, q=16, i8s=False):
    # the FP64 arm must be the FP64 kernel itself, not "auto" (which picks the
    # int8 scatter for large dense node sets)
    return sgl.plan(B, pts, rho=rho, q=q, profile=True, backend="i8" if i8s else "tiled")


gd = os.path.join(ROOT, "tests", "golden")
for name in ["ref_b12_q12.npz", "ref_b8_q16.npz", "ref_cfg1.npz", "ref_cfg2_sub2000.npz", "ref_cfg3_sub600.npz",
             "ref_edges_b8_q16.npz", "ref_b4_q8.npz"]:
    g = np.load(os.path.join(gd, name))
    if "adj" not in g:
        continue
    B, q, rho = int(g["B"]), int(g["q"]), float(g["rho"])
    try:
        p8 = mk(B, g["points"], rho, q, True)
        p6 = mk(B, g["points"], rho, q, False)
        a8 = sgl.adjoint(p8, g["values"])
        a6 = sgl.adjoint(p6, g["values"])
        print(f"{name}: B={B} q={q} M={p8.m_points} i8s vs ref {rel(a8, g['adj']):.2e}  fp64 vs ref "
              f"{rel(a6, g['adj']):.2e}  i8s vs fp64 {rel(a8, a6):.2e}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name}: ERROR {e}", flush=True)

for cfg, M in [(3, 1_000_000), (3, 10_000_000), (2, None), (4, 10_000_000)]:
    w = workloads.config(cfg, M=M)
    out = {}
    for i8s in (False, True):
        p = mk(w.B, w.points, w.rho, 16, i8s)
        a = sgl.adjoint(p, w.values)
        ms = []
        for _ in range(3):
            a = sgl.adjoint(p, w.values)
            ms.append(p.stage_ms("adjoint")["window"])
        out[i8s] = (a, min(ms))
        p.close()
    print(f"cfg{cfg} M={w.M}: scatter fp64 {out[False][1]:.3f} ms  i8 {out[True][1]:.3f} ms "
          f"(x{out[False][1] / out[True][1]:.2f})  i8 vs fp64 rel-linf {rel(out[True][0], out[False][0]):.2e}",
          flush=True)
