"""Plan construction time at a BASELINE config, with the per-stage breakdown
(SGL_FLAG_I8_PROF prints it to stderr); device-resident points, warm context."""
import argparse, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import _native, workloads
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--m", type=int, default=None)
a = ap.parse_args()
w = workloads.config(a.config, M=a.m)
pts = torch.as_tensor(w.points, device="cuda")
sgl.plan(w.B, pts[:1000])   # context + module load
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = sgl.plan(w.B, pts, flags=_native.FLAG_I8_PROF if rep else 0)
    torch.cuda.synchronize()
    print(f"rep {rep}: plan {time.perf_counter() - t0:.3f} s (plan_ms {p.stats['plan_ms']:.1f})", flush=True)
    p.close()
