"""Seeded synthetic inputs with the reference's draw order.

Restates the reference generators (`generate.py:17-75` in `sglnufft`) so the
benchmark and tests build exactly the BASELINE.json inputs: numpy PCG64
streams, coefficients as one real block then one imaginary block, ball
points as radii / cosines / azimuths.  Pinned against the reference outputs
in `tests/golden/` (`tests/test_generate.py`).
"""
from __future__ import annotations

import numpy as np


def coeff_count(B: int) -> int:
    """Number of (n, l, m) triples with n <= B (indexing.py:22-26)."""
    if B < 1:
        raise ValueError("bandwidth must be >= 1")
    return B * (B + 1) * (2 * B + 1) // 6


def nlm_table(B: int) -> np.ndarray:
    """(count, 3) int64 rows (n, l, m) in mu order, mu = n(n-1)(2n-1)/6 +
    l(l+1) + m (indexing.py:41-81)."""
    rows = [(n, l, m) for n in range(1, B + 1) for l in range(n) for m in range(-l, l + 1)]
    return np.array(rows, dtype=np.int64).reshape(-1, 3)


def rng_from(seed) -> np.random.Generator:
    """PCG64 generator, or pass-through of an existing one (generate.py:17-20)."""
    if isinstance(seed, np.random.Generator):
        return seed
    return np.random.Generator(np.random.PCG64(seed))


def gen_coeffs(B: int, seed) -> np.ndarray:
    """complex128 coefficients, Re then Im blocks of U[-1,1] (generate.py:23-32)."""
    g = rng_from(seed)
    n = coeff_count(B)
    re = g.uniform(-1.0, 1.0, n)
    im = g.uniform(-1.0, 1.0, n)
    return re + 1j * im


def gen_points_ball(M: int, kappa: float, seed) -> np.ndarray:
    """Volume-uniform ball points as (r, theta, phi) rows (generate.py:35-49)."""
    if M < 1:
        raise ValueError("need at least one point")
    if kappa <= 0:
        raise ValueError("ball radius must be positive")
    g = rng_from(seed)
    r = kappa * g.random(M) ** (1.0 / 3.0)
    ct = g.uniform(-1.0, 1.0, M)
    phi = g.uniform(0.0, 2.0 * np.pi, M)
    return np.column_stack([r, np.arccos(ct), phi])


def cartesian_to_spherical(xyz: np.ndarray) -> np.ndarray:
    """(..., 3) Cartesian -> (r, theta, phi), phi in [0, 2 pi) (generate.py:67-75)."""
    xyz = np.asarray(xyz, dtype=float)
    r = np.linalg.norm(xyz, axis=-1)
    safe = np.where(r > 0, r, 1.0)
    ct = np.where(r > 0, xyz[..., 2] / safe, 1.0)
    theta = np.arccos(np.clip(ct, -1.0, 1.0))
    phi = np.mod(np.arctan2(xyz[..., 1], xyz[..., 0]), 2.0 * np.pi)
    return np.stack([r, theta, phi], axis=-1)


def gen_grid(N: int, kappa: float) -> np.ndarray:
    """N^3 Cartesian grid kappa (2j/N - 1), axis 0 slowest (generate.py:52-64)."""
    if N < 1:
        raise ValueError("grid extent must be >= 1")
    if kappa <= 0:
        raise ValueError("kappa must be positive")
    g = kappa * (2.0 * np.arange(N) / N - 1.0)
    x, y, z = np.meshgrid(g, g, g, indexing="ij")
    return cartesian_to_spherical(np.column_stack([x.ravel(), y.ravel(), z.ravel()]))
