import numpy as np, sys
import paper_1809_10786_b200 as sgl
sys.path.insert(0, '.')
from oracle import sgl_oracle as o
def case(seed):
    rng = np.random.default_rng(10_000 + seed)
    B = int(rng.integers(1, 33)); sigma = int(rng.choice([2, 2, 2, 3])); q = int(rng.integers(2, 17))
    if q >= 4 * sigma * B: q = max(1, 4 * sigma * B - 1)
    M = int(rng.choice([1, 7, 100, 3000, 50_000, 200_000])); kind = int(rng.integers(0, 4))
    if kind == 0: pts = sgl.gen_points_ball(M, float(rng.uniform(0.5, 8.0)), rng)
    elif kind == 1: pts = sgl.cartesian_to_spherical(rng.normal(0, np.sqrt(0.5), (M, 3)))
    elif kind == 2:
        g = max(2, int(round(M ** (1 / 3)))); pts = sgl.gen_grid(g, float(rng.uniform(1.0, 6.0)))
    else:
        pts = np.column_stack([np.full(M, 1.0), rng.choice([0.0, np.pi / 2, np.pi], M), rng.choice([0.0, np.pi / 2, np.pi, 1.5 * np.pi], M)])
    compact = bool(rng.random() < 0.2)
    c = sgl.gen_coeffs(B, rng); v = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    return B, sigma, q, compact, pts, c, v
rel = lambda x, y: float(np.max(np.abs(x - y)) / np.max(np.abs(y)))
for seed in [int(s) for s in (sys.argv[1:] or ["578", "702", "2311", "1634"])]:
    B, sigma, q, compact, pts, c, v = case(seed)
    pa = sgl.plan(B, pts, sigma=sigma, q=q, compact_k1=compact, backend="tiled")
    pb = sgl.plan(B, pts, sigma=sigma, q=q, compact_k1=compact, backend="generic")
    op = o.oracle_plan(B, pts, sigma=sigma, q=q, compact_k1=compact)
    fo, ao = o.oracle_forward(op, c), o.oracle_adjoint(op, v)
    print(seed, B, sigma, q, len(pts), pa.nfft.grid_shape, "tiled fwd/adj vs oracle", rel(sgl.forward(pa, c), fo), rel(sgl.adjoint(pa, v), ao),
          "generic", rel(sgl.forward(pb, c), fo), rel(sgl.adjoint(pb, v), ao), "tiles", pa.stats["n_tiles"])
