"""Guard estimates vs measured int8-vs-FP64 error at full size (configs 3, 4)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import _native, workloads

def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))

for cfg in (3, 4):
    w = workloads.config(cfg)
    t0 = time.time()
    p8 = sgl.plan(w.B, w.points, flags=_native.FLAG_NO_GUARD)
    print(f"cfg{cfg} plan {time.time() - t0:.2f}s stats {p8.stats}", flush=True)
    a8 = sgl.adjoint(p8, w.values)
    g = p8.guard
    f8 = sgl.forward(p8, w.coeffs) if cfg == 3 else None
    g2 = p8.guard
    p8.close()
    p64 = sgl.plan(w.B, w.points, backend="tiled")
    a64 = sgl.adjoint(p64, w.values)
    print(f"cfg{cfg} adj err {rel(a8, a64):.3e} est {g['est_adj']:.3e}", flush=True)
    if f8 is not None:
        f64 = sgl.forward(p64, w.coeffs)
        print(f"cfg{cfg} fwd err {rel(f8, f64):.3e} est {g2['est_fwd']:.3e}", flush=True)
    p64.close()
    del w
