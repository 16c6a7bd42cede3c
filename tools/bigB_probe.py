"""Large-bandwidth smoke: plan + forward + adjoint + pairing at B = 192
(oversampled grid 2048 x 2048 x 1024, 72 GB with the halo)."""
import sys
import time

import numpy as np
import torch

import paper_1809_10786_b200 as sgl

B = int(sys.argv[1]) if len(sys.argv) > 1 else 192
rng = np.random.default_rng(0)
pts = sgl.gen_points_ball(4000, 20.0, rng)
c = sgl.gen_coeffs(B, rng) / np.repeat(np.arange(1, B + 1), [n * n for n in range(1, B + 1)])
v = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
t0 = time.time()
p = sgl.plan(B, pts, profile=True)
t1 = time.time()
f = sgl.forward(p, c)
a = sgl.adjoint(p, v)
torch.cuda.synchronize()
lhs, rhs = np.vdot(v, f), np.vdot(a, c)
free, total = torch.cuda.mem_get_info()
print(f"B={B} grid={p.nfft.grid_shape} plan {t1 - t0:.1f} s, fwd {p.stage_ms('forward')}, adj {p.stage_ms('adjoint')}")
print(f"pairing rel {abs(lhs - rhs) / (np.linalg.norm(f) * np.linalg.norm(v)):.2e}, finite {np.all(np.isfinite(f))} "
      f"{np.all(np.isfinite(a))}, device memory used {(total - free) / 1e9:.1f} GB")
