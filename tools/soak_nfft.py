"""Soak test of the NFFT layer: random d, n, per-axis sigma, q and node sets
(incl. nodes outside [0, 2 pi) and on grid lines); tiled vs per-node kernels
(d = 3) and fast vs exact within the reference's error bound."""
import sys
import time

import numpy as np

import paper_1809_10786_b200 as sgl

n_plans = int(sys.argv[1]) if len(sys.argv) > 1 else 300
worst_kern, worst_bound = 0.0, 0.0
t0 = time.time()
for seed in range(n_plans):
    rng = np.random.default_rng(30_000 + seed)
    d = int(rng.choice([1, 2, 3, 3, 3]))
    n = tuple(int(2 * rng.integers(1, 17)) for _ in range(d))
    sig = tuple(int(rng.choice([2, 2, 3, 4])) for _ in range(d))
    grid = [1 << int(np.ceil(np.log2(s * k))) for s, k in zip(sig, n)]
    q = int(rng.integers(1, min(17, min(grid))))
    M = int(rng.choice([1, 50, 2000, 30_000]))
    if rng.random() < 0.3:   # nodes on grid lines of the oversampled grid
        nodes = np.stack([2 * np.pi * rng.integers(0, g, M) / g for g in grid], axis=1)
    else:
        nodes = rng.uniform(-2.0, 2 * np.pi + 2.0, (M, d))
    f = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    v = rng.uniform(-1, 1, M) + 1j * rng.uniform(-1, 1, M)
    pa = sgl.nfft_plan(d, n, sig, q, nodes)
    fa, aa = sgl.nfft_execute(pa, f), sgl.nfft_adjoint_execute(pa, v)
    if d == 3:
        pb = sgl.nfft_plan(d, n, sig, q, nodes, backend="generic")
        for x, y in ((fa, sgl.nfft_execute(pb, f)), (aa, sgl.nfft_adjoint_execute(pb, v))):
            r = float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))
            worst_kern = max(worst_kern, r)
            if r > 1e-11:
                print("KERNEL MISMATCH", seed, d, n, sig, q, M, r)
        pb.close()
    if M <= 2000 and np.prod(n) <= 4096:
        ex = sgl.ndft(d, n, f, nodes)
        err = float(np.max(np.abs(fa - ex)))
        bound = sgl.nfft_error_bound(d, min(sig), q, float(np.sum(np.abs(f)))) if min(sig) >= (np.sqrt(d) + 1) / 2 \
            else np.inf
        bound += 1e-13 * float(np.sum(np.abs(f)))   # round-off allowance (the reference's tests allow one too)
        ratio = err / bound if bound > 0 else 0.0
        worst_bound = max(worst_bound, ratio)
        if ratio > 1.0:
            print("BOUND EXCEEDED", seed, d, n, sig, q, M, err, bound)
    pa.close()
print(f"{n_plans} random NFFT plans: worst tiled-vs-generic {worst_kern:.2e}, worst error / bound {worst_bound:.3f}, "
      f"{time.time() - t0:.0f} s")
