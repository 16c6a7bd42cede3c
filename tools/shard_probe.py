"""Per-rank work of config 3 strong scaling at N ranks, measured one rank at a
time on one GPU: contiguous shards of the caller order (random subsamples, 1/N
of the node density) against radial shells of equal node count (full density:
`distributed.shard_indices(..., "radial")`).  Device ms of one forward +
adjoint per rank (window stages and total).  PYTHONPATH=. python tools/shard_probe.py [N]"""
import sys

import numpy as np
import torch

import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import workloads
from paper_1809_10786_b200.distributed import shard_indices

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = workloads.config(3)
c = torch.as_tensor(w.coeffs, device="cuda")
for mode in (sys.argv[2:] or ["contiguous", "radial", "theta"]):
    tot, win = [], []
    for k in range(N):
        idx = shard_indices(w.points, k, N, mode)
        p = sgl.plan(w.B, w.points[idx], rho=w.rho, profile=True)
        v = torch.as_tensor(w.values[idx], device="cuda")
        for _ in range(3):
            sgl.forward(p, c), sgl.adjoint(p, v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sgl.forward(p, c), sgl.adjoint(p, v)
        e1.record()
        torch.cuda.synchronize()
        sgl.forward(p, c), sgl.adjoint(p, v)
        torch.cuda.synchronize()
        tot.append(e0.elapsed_time(e1) / 5)
        win.append((p.stage_ms("forward")["window"], p.stage_ms("adjoint")["window"]))
        p.close()
    print(f"{mode:10s} N={N}: per-rank fwd+adj ms " + " ".join(f"{t:.2f}" for t in tot) +
          f" | max {max(tot):.2f} (window gather/scatter of the slowest: {win[int(np.argmax(tot))][0]:.2f} / "
          f"{win[int(np.argmax(tot))][1]:.2f}); strong-scaling efficiency bound {53.5 / (N * max(tot)):.2f}",
          flush=True)
