"""int8 vs FP64 scatter across node densities of the config-3 distribution
(random subsamples = the node shards of a strong-scaling run): adjoint window
stage ms for backend i8 and tiled, the plan's int8 K-steps per node, the
automatic choice, and the accuracy guard's estimate / fallbacks for the int8
engine.  PYTHONPATH=. python tools/scatter_crossover.py"""
import sys

import numpy as np
import torch

import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import workloads

full = workloads.config(3)
for M in [int(x) for x in (sys.argv[1:] or [156250, 312500, 625000, 1250000, 2500000, 5000000])]:
    pts, vals = full.points[:M], full.values[:M]
    v = torch.as_tensor(vals, device="cuda")
    res = {}
    for b in ("i8", "tiled", "auto"):
        p = sgl.plan(full.B, pts, rho=full.rho, backend=b, profile=True)
        for _ in range(3):
            sgl.adjoint(p, v)
        torch.cuda.synchronize()
        ms = []
        for _ in range(5):
            sgl.adjoint(p, v)
            torch.cuda.synchronize()
            ms.append(p.stage_ms("adjoint")["window"])
        st, gd = p.stats, p.guard
        res[b] = (float(np.median(ms)), st["i8_sksteps"], st["i8_scatter"], gd["est_adj"], gd["adj_fallbacks"])
        p.close()
    i8, tl, au = res["i8"], res["tiled"], res["auto"]
    print(f"M={M:9d}: int8 {i8[0]:7.3f} ms (K-steps/node {i8[1] / M:.3f}, guard est {i8[3]:.2e}, fallbacks {i8[4]}), "
          f"FP64 {tl[0]:7.3f} ms, auto picks {'int8' if au[2] else 'FP64'} ({au[0]:.3f} ms)", flush=True)
