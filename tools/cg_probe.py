"""Per-iteration cost of the device CG inverse on small systems: the eager
loop (host-read step sizes) against the CUDA-graph loop, and the bare
forward + adjoint pair of the same plan.  PYTHONPATH=. python tools/cg_probe.py"""
import time

import numpy as np
import torch

import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import solvers

for B, N, q in [(4, 20, 8), (8, 25, 15), (16, 50, 16), (32, 80, 16)]:
    pts = sgl.gen_grid(N, 3.0)
    c = sgl.gen_coeffs(B, 1)
    vals = sgl.evaluate_direct(c, B, pts)
    res = {}
    for graph in (False, True):
        solvers.invert(pts, vals, B, q=q, max_iter=5, tol=0.0, graph=graph)   # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = solvers.invert(pts, vals, B, q=q, max_iter=200, tol=0.0, graph=graph)
        torch.cuda.synchronize()
        res[graph] = (time.perf_counter() - t0, rep)
    a, b = res[False][1], res[True][1]
    assert a.iterations == b.iterations == 200
    p = sgl.plan(B, pts, q=q)
    op = solvers.operator_from_plan(p)
    tcap = {}
    for graph in (False, True):   # the iterations alone: one plan, 20 vs 220 iterations
        ts = []
        for m in (20, 220):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            solvers.cgnr(op, vals, max_iter=m, tol=0.0, graph=graph)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        tcap[graph] = (ts[1] - ts[0]) / 200
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
    print(f"B={B} M={len(pts)}: CG iteration eager {1e3 * tcap[False]:.3f} ms, graph {1e3 * tcap[True]:.3f} ms; "
          f"invert(200 it, incl. plan and capture) eager {res[False][0]:.3f} s, graph {res[True][0]:.3f} s; "
          f"bare fwd+adj pair {1e3 * t2 / 200:.3f} ms")
