"""Basis indexing of the SGL expansion (reference indexing.py:22-81).

mu(n, l, m) = n(n-1)(2n-1)/6 + l(l+1) + m for 1 <= n <= B, 0 <= l < n,
|m| <= l: the coefficient order of `forward` / `adjoint`.
"""
from __future__ import annotations

from typing import NamedTuple

import numpy as np

from .generate import coeff_count, nlm_table


class SglIndex(NamedTuple):
    """Basis triple (n, l, m) with |m| <= l < n."""
    n: int
    l: int
    m: int


def _tetra(n: int) -> int:
    return n * (n - 1) * (2 * n - 1) // 6


def nlm_to_mu(n: int, l: int, m: int) -> int:
    """Linear storage index of (n, l, m)."""
    if not (0 <= l < n and abs(m) <= l):
        raise ValueError(f"invalid triple ({n}, {l}, {m})")
    return _tetra(n) + l * (l + 1) + m


def mu_to_nlm(mu: int, B: int) -> SglIndex:
    """Inverse of `nlm_to_mu` on [0, coeff_count(B)) by integer search."""
    mu = int(mu)
    if not (0 <= mu < coeff_count(B)):
        raise ValueError(f"mu = {mu} out of range for B = {B}")
    lo, hi = 1, B                      # largest n with tetra(n) <= mu
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if _tetra(mid) <= mu:
            lo = mid
        else:
            hi = mid - 1
    rem = mu - _tetra(lo)
    l = int(np.sqrt(rem))
    while l * l > rem:
        l -= 1
    while (l + 1) * (l + 1) <= rem:
        l += 1
    return SglIndex(lo, l, rem - l * (l + 1))


def mu_to_nlm_array(B: int) -> np.ndarray:
    """(count, 3) int64 table of (n, l, m) in mu order."""
    return nlm_table(B)
