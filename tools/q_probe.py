"""Window-kernel time versus the cutoff q (config-3 shape, 2e6 nodes)."""
import numpy as np
import torch

import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import workloads

w = workloads.config(3, M=2_000_000)
cd = torch.as_tensor(w.coeffs, device="cuda")
vd = torch.as_tensor(w.values, device="cuda")
pts = torch.as_tensor(w.points, device="cuda")
for q in (4, 8, 12, 16):
    p = sgl.plan(w.B, pts, q=q, rho=w.rho, profile=True)
    for _ in range(3):
        sgl.forward(p, cd)
        sgl.adjoint(p, vd)
    torch.cuda.synchronize()
    g, s = p.stage_ms("forward")["window"], p.stage_ms("adjoint")["window"]
    flop = 4.0 * (2 * q) ** 3 * w.M / 1e12
    print(f"q={q:2d} gather {g:7.3f} ms ({flop / (g * 1e-3) / 37.1:.2f} of FP64 peak)  "
          f"scatter {s:7.3f} ms ({flop / (s * 1e-3) / 37.1:.2f})  box {p._info.n_tiles} tiles")
    p.close()
