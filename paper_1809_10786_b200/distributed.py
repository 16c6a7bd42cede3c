"""Multi-GPU NFSGLFT: node shards over a torch.distributed group.

One process per GPU.  The forward transform is pointwise in the nodes, so a
rank evaluates its own shard with no collective (the oversampled grid is
rebuilt per rank: basal stage + FFT cost ~1.6 ms at B=64, less than moving the
1.07 GB grid over NVLink).  The adjoint is a sum over nodes, so each rank runs
the full adjoint of its shard and the ranks all-reduce the coefficient vector
(count complex128: 1.4 MB at B=64, 11 MB at B=128) over NCCL.  That single
small all-reduce replaces the grid reduce-scatter + transposes a slab-
decomposed FFT would need (8.6 GB at B=128).  The radial parameter rho must
be global (transform.py:39-43, 345-348): it is the all-reduce max of the
shards' radii unless the caller pins it.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np


def shard_bounds(M: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, count-balanced [start, stop) of rank's shard."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(M, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


@dataclass
class Compute:
    """The per-rank transform implementation (default: this package's CUDA path)."""
    plan: Callable
    forward: Callable
    adjoint: Callable


def cuda_compute() -> Compute:
    from . import transform
    return Compute(transform.plan, transform.forward, transform.adjoint)


def _dist():
    import torch.distributed as dist
    return dist


def _reduce_(arr, op: str, group=None):
    """In-place all-reduce of a numpy array or torch tensor (complex: as real pairs)."""
    import torch
    dist = _dist()
    rop = dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM
    backend = dist.get_backend(group)
    if isinstance(arr, torch.Tensor):
        t = torch.view_as_real(arr) if arr.is_complex() else arr
        dist.all_reduce(t, op=rop, group=group)
        return arr
    host = torch.from_numpy(np.ascontiguousarray(arr))
    t = host.cuda() if backend == "nccl" else host
    dist.all_reduce(torch.view_as_real(t) if t.is_complex() else t, op=rop, group=group)
    return t.cpu().numpy() if t is not host else host.numpy()


def global_rho(local_points, group=None) -> float:
    """choose_rho over the union of all shards (transform.py:39-43)."""
    pts = local_points
    if type(pts).__module__.startswith("torch"):
        r = float(pts[:, 0].max().item()) if pts.shape[0] else 0.0
    else:
        pts = np.atleast_2d(np.asarray(pts, dtype=float))
        r = float(np.max(pts[:, 0])) if pts.size else 0.0
    r = float(_reduce_(np.array([r]), "max", group)[0])
    return r if r > 0 else 1.0


class ShardedPlan:
    """This rank's plan over its node shard; `adjoint` returns the global
    coefficient vector (identical on every rank)."""

    def __init__(self, B: int, local_points, *, group=None, rho: float | None = None,
                 compute: Compute | None = None, **plan_kw):
        self.group = group
        self.compute = compute or cuda_compute()
        self.rho = float(rho) if rho is not None else global_rho(local_points, group)
        self.plan = self.compute.plan(B, local_points, rho=self.rho, **plan_kw)

    def forward(self, coeffs):
        """Values at this rank's nodes (no collective)."""
        return self.compute.forward(self.plan, coeffs)

    def adjoint(self, local_values):
        """sum over all ranks of the shard adjoints (one all-reduce)."""
        return _reduce_(self.compute.adjoint(self.plan, local_values), "sum", self.group)
