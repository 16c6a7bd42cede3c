"""The five BASELINE.json configurations as seeded synthetic inputs.

Draw order follows SURVEY.md section 8(d): coefficients first
(`gen_coeffs`), then nodes, then the adjoint's node values (real block, then
imaginary block, each U[-1, 1]).  Nodes given in Cartesian form are converted
with the reference's `cartesian_to_spherical`.  No public dataset exists for
this path; these seeded inputs are the whole specification.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .generate import (cartesian_to_spherical, coeff_count, gen_coeffs, gen_grid,
                       gen_points_ball, rng_from)


@dataclass
class Workload:
    name: str
    B: int
    points: np.ndarray          # (M, 3) spherical (r, theta, phi)
    coeffs: np.ndarray          # (count,) or (K, count) complex128
    values: np.ndarray | None   # (M,) complex128 adjoint input
    rho: float                  # max radius of the FULL node set
    directions: str             # "fwd", "fwd+adj" or "adj"

    @property
    def M(self) -> int:
        return self.points.shape[0]


def _values(rng, M):
    re = rng.uniform(-1.0, 1.0, M)
    im = rng.uniform(-1.0, 1.0, M)
    return re + 1j * im


def _rho(points):
    r = float(np.max(points[:, 0]))
    return r if r > 0 else 1.0


def config(idx: int, M: int | None = None, seed: int = 0) -> Workload:
    """Build BASELINE config `idx` (1-based).  `M` overrides the node count
    (the distribution is unchanged; for config 2 the 100^3 grid is fixed)."""
    rng = rng_from(seed)
    if idx == 1:
        B = 16
        M = 20_000 if M is None else M
        c = gen_coeffs(B, rng)
        pts = cartesian_to_spherical(rng.normal(0.0, np.sqrt(0.5), (M, 3)))
        return Workload("cfg1_B16_normal", B, pts, c, _values(rng, M), _rho(pts), "fwd")
    if idx == 2:
        B = 32
        c = gen_coeffs(B, rng)
        pts = gen_grid(100, 4.0)
        return Workload("cfg2_B32_grid100", B, pts, c, _values(rng, pts.shape[0]), _rho(pts), "fwd+adj")
    if idx == 3:
        B = 64
        M = 10_000_000 if M is None else M
        c = gen_coeffs(B, rng)
        n_of_mu = np.concatenate([np.full(n * n, n) for n in range(1, B + 1)])
        c = c / n_of_mu
        pts = gen_points_ball(M, 16.0, rng)
        return Workload("cfg3_B64_ball16", B, pts, c, _values(rng, M), _rho(pts), "fwd+adj")
    if idx == 4:
        B = 128
        M = 100_000_000 if M is None else M
        c = gen_coeffs(B, rng)
        h = M // 2
        a = cartesian_to_spherical(rng.normal(0.0, np.sqrt(0.5), (h, 3)))
        b = gen_points_ball(M - h, 22.0, rng)
        pts = np.concatenate([a, b])[rng.permutation(M)]
        return Workload("cfg4_B128_mixed", B, pts, c, _values(rng, M), _rho(pts), "adj")
    if idx == 5:
        B = 48
        M = 2_000_000 if M is None else M
        c = np.stack([gen_coeffs(B, rng) for _ in range(64)])
        pts = cartesian_to_spherical(rng.normal(0.0, np.sqrt(0.5), (M, 3)))
        return Workload("cfg5_B48_batch64", B, pts, c, None, _rho(pts), "fwd")
    raise ValueError(f"unknown config {idx}")


def subset(w: Workload, k: int, seed: int = 1) -> tuple[np.ndarray, Workload]:
    """Seeded k-node subset with rho pinned to the full set's."""
    if k >= w.M:
        return np.arange(w.M), w
    sel = np.sort(np.random.Generator(np.random.PCG64(seed)).choice(w.M, k, replace=False))
    vals = None if w.values is None else w.values[sel]
    return sel, Workload(w.name + f"_sub{k}", w.B, w.points[sel], w.coeffs, vals, w.rho, w.directions)


assert coeff_count(16) == 1496
