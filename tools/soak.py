"""Soak test: many random plans (B, sigma, q, node distributions up to 2e5
nodes), tiled kernels against the per-node kernels, forward and adjoint.
Prints the worst relative difference; any hang trips the ring watchdog."""
import sys
import time

import numpy as np

import paper_1809_10786_b200 as sgl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
# second argument: the backend under test ("tiled": FP64 DMMA kernels; "auto":
# the int8 tensor-core gather + FP64 scatter), always against the per-node kernels
backend = sys.argv[2] if len(sys.argv) > 2 else "tiled"
worst = 0.0
t0 = time.time()
for seed in range(n):
    rng = np.random.default_rng(10_000 + seed)
    B = int(rng.integers(1, 33))
    sigma = int(rng.choice([2, 2, 2, 3]))
    q = int(rng.integers(2, 17))
    if q >= 4 * sigma * B:
        q = max(1, 4 * sigma * B - 1)
    M = int(rng.choice([1, 7, 100, 3000, 50_000, 200_000]))
    kind = int(rng.integers(0, 4))
    if kind == 0:
        pts = sgl.gen_points_ball(M, float(rng.uniform(0.5, 8.0)), rng)
    elif kind == 1:
        pts = sgl.cartesian_to_spherical(rng.normal(0, np.sqrt(0.5), (M, 3)))
    elif kind == 2:
        g = max(2, int(round(M ** (1 / 3))))
        pts = sgl.gen_grid(g, float(rng.uniform(1.0, 6.0)))
    else:
        pts = np.column_stack([np.full(M, 1.0), rng.choice([0.0, np.pi / 2, np.pi], M),
                               rng.choice([0.0, np.pi / 2, np.pi, 1.5 * np.pi], M)])
    compact = bool(rng.random() < 0.2)
    c = sgl.gen_coeffs(B, rng)
    v = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    pa = sgl.plan(B, pts, sigma=sigma, q=q, compact_k1=compact, backend=backend if q <= 16 else "auto")
    pb = sgl.plan(B, pts, sigma=sigma, q=q, compact_k1=compact, backend="generic")
    for x, y in ((sgl.forward(pa, c), sgl.forward(pb, c)), (sgl.adjoint(pa, v), sgl.adjoint(pb, v))):
        den = np.max(np.abs(y))
        r = float(np.max(np.abs(x - y)) / den) if den > 0 else float(np.max(np.abs(x)))
        worst = max(worst, r)
        if not r <= 1e-11:
            print("MISMATCH", seed, B, sigma, q, M, kind, compact, r)
    pa.close()
    pb.close()
print(f"{n} random plans, worst {backend}-vs-generic rel-linf {worst:.2e}, {time.time() - t0:.0f} s")
