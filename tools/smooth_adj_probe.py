"""Which engine is off on smooth adjoint inputs (v = exp(-r^2), B = 32)?
int8 scatter, FP64 tiled scatter, per-node FP64 kernels and the CPU oracle."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1809_10786_b200 as sgl
from oracle import sgl_oracle as o
import subprocess
subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)

def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))

rng = np.random.default_rng(0)
for B, M in [(32, 20000), (32, 4000), (16, 20000)]:
    rad = 2.0 + B / 8
    pts = sgl.gen_points_ball(M, rad, rng)
    v = np.exp(-pts[:, 0] ** 2).astype(complex)
    out = {}
    for be in ("i8", "tiled", "generic"):
        p = sgl.plan(B, pts, backend=be)
        out[be] = sgl.adjoint(p, v)
    op = o.oracle_plan(B, pts)
    out["oracle"] = o.oracle_adjoint(op, v)
    for k in ("i8", "tiled", "generic"):
        print(f"B={B} M={M} {k:8s} vs oracle {rel(out[k], out['oracle']):.2e}  vs generic {rel(out[k], out['generic']):.2e}",
              flush=True)
    mag = np.abs(out["oracle"])
    print("  |c| max", mag.max(), "median", np.median(mag), "argmax", int(np.argmax(np.abs(out['i8'] - out['tiled']))),
          flush=True)
