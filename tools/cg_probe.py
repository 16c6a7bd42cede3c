"""Per-iteration cost of the device CG inverse on small systems (latency probe)."""
import time

import numpy as np
import torch

import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import solvers

for B, N, q in [(4, 20, 8), (8, 25, 15), (16, 50, 16)]:
    pts = sgl.gen_grid(N, 3.0)
    c = sgl.gen_coeffs(B, 1)
    vals = sgl.evaluate_direct(c, B, pts)
    solvers.invert(pts, vals, B, q=q, max_iter=5, tol=0.0)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = solvers.invert(pts, vals, B, q=q, max_iter=200, tol=0.0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    p = sgl.plan(B, pts, q=q)
    cd = torch.as_tensor(c, device="cuda")
    vd = torch.as_tensor(vals, device="cuda")
    for _ in range(3):
        sgl.forward(p, cd); sgl.adjoint(p, vd)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(200):
        sgl.forward(p, cd); sgl.adjoint(p, vd)
    torch.cuda.synchronize()
    t2 = time.perf_counter() - t1
    print(f"B={B} M={len(pts)}: invert {rep.iterations} it in {t:.3f} s = {1e3 * t / max(rep.iterations, 1):.3f} ms/it; "
          f"fwd+adj pair {1e3 * t2 / 200:.3f} ms")
