"""Config-4 golden subset against the extended-precision truth: default plan,
FP64 tiled kernels, precise_tables (basal matrices built in x87 80-bit)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1809_10786_b200 as sgl
from conftest import load_golden

def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))

g, t = load_golden("cfg4_sub120"), load_golden("cfg4_truth")
print("reference fast vs truth", float(t["ref_fast_err"]))
for kw in ({}, {"backend": "tiled"}, {"precise_tables": True}):
    t0 = time.time()
    p = sgl.plan(128, g["points"], rho=float(g["rho"]), **kw)
    dt = time.time() - t0
    a = sgl.adjoint(p, g["values"])
    err = np.abs(a - t["truth"]) / np.max(np.abs(t["truth"]))
    print(kw, f"plan {dt:.2f}s  vs truth {rel(a, t['truth']):.3e}  vs ref {rel(a, g['adj']):.3e}  argmax mu {int(np.argmax(err))}",
          flush=True)
