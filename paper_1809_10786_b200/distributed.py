"""Multi-GPU NFSGLFT: node shards over a torch.distributed group.

One process per GPU.  The reference has no multi-GPU code; the
partition follows BASELINE's north star:

* forward (pointwise in the nodes): each rank evaluates its own node shard;
  the oversampled grid is rebuilt per rank (basal stage + FFT, ~1.6 ms at
  B = 64), cheaper than moving the 1.07 GB grid.  No collective.
* adjoint (a sum over nodes), two partitions:
  - ``partition="grid"`` (the north star's): each rank spreads its shard into
    its own oversampled grid; an NCCL reduce-scatter over axis-0 plane blocks
    combines the grids; each rank runs the 2-D FFT (axes 1-2) of its planes
    and packs the spectral box the basal stage reads (1/4.8 of a plane at
    B = 64); the packed planes are gathered to rank 0, which runs the 1-D FFT
    along axis 0, crop, deconvolution and basal adjoint and broadcasts the
    coefficients.  (The 1-D FFT over the packed planes is ~0.1 ms, so a
    gather replaces the all-to-all + distributed 1-D FFT of SURVEY 8(e).)
  - ``partition="coeffs"``: each rank runs the whole adjoint of its shard and
    the ranks all-reduce the coefficient vector (1.4 MB at B = 64, 11 MB at
    B = 128).  The FFT and basal adjoint are linear, so reducing after them is
    exact; the FFT is replicated instead of split.
  ``partition="auto"`` picks by the bytes/time model `partition_model`
  (DESIGN.md section 6): on NVSwitch the grid reduce-scatter (1.1 GB at B = 64,
  9.4 GB at B = 128) costs more than the replicated FFT it saves, so "auto"
  is "coeffs" for the BASELINE configurations.
* rho must be global (transform.py:39-43, 345-348): the all-reduce max of
  the shards' radii unless the caller pins it.
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
    """The per-rank transform implementation (default: this package's CUDA
    path).  The grid partition also needs the stage functions:
    ``spread(plan, values) -> grid``, ``grid_info(plan) -> (N0, crop1, crop2)``,
    ``slab_fft(plan, grid, a0, a1) -> packed (a1-a0, crop1, crop2)``,
    ``from_packed(plan, packed_all) -> coeffs``; ``grid`` is a torch tensor
    viewed as (N0, plane) or whatever the stage functions agree on."""
    plan: Callable
    forward: Callable
    adjoint: Callable
    spread: Callable | None = None
    grid_info: Callable | None = None
    slab_fft: Callable | None = None
    from_packed: Callable | None = None


def _torch():
    import torch
    return torch


class _DeviceArray:
    """__cuda_array_interface__ view of library-owned device memory (zero copy)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str = "<c16"):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def cuda_compute() -> Compute:
    from . import _native, transform

    def grid_info(p):
        gi = _native.GridInfo()
        _native.check(_native.lib().sgl_plan_grid(p._handle, gi))
        return gi

    def spread(p, values):
        torch = _torch()
        dev = torch.device("cuda", p.device)
        v = torch.as_tensor(values, device=dev).to(torch.complex128).contiguous()
        if tuple(v.shape) != (p.m_points,):
            raise ValueError("values length does not match the plan")
        st = torch.cuda.current_stream(dev).cuda_stream
        _native.check(_native.lib().sgl_adjoint_spread(p._handle, v.data_ptr() if v.numel() else None, st))
        gi = grid_info(p)
        return torch.as_tensor(_DeviceArray(gi.data, (gi.N0, gi.plane_elems)), device=dev)

    def slab_fft(p, grid, a0, a1):
        torch = _torch()
        gi = grid_info(p)
        dev = torch.device("cuda", p.device)
        out = torch.empty((a1 - a0, gi.crop1, gi.crop2), dtype=torch.complex128, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _native.check(_native.lib().sgl_adjoint_slab_fft(p._handle, int(a0), int(a1),
                                                         out.data_ptr() if out.numel() else None, st))
        return out

    def from_packed(p, packed):
        torch = _torch()
        dev = torch.device("cuda", p.device)
        out = torch.empty((p.count,), dtype=torch.complex128, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _native.check(_native.lib().sgl_adjoint_from_packed(p._handle, packed.contiguous().data_ptr(),
                                                            out.data_ptr(), st))
        return out

    return Compute(transform.plan, transform.forward, transform.adjoint, spread=spread,
                   grid_info=lambda p: (lambda g: (g.N0, g.crop1, g.crop2))(grid_info(p)),
                   slab_fft=slab_fft, from_packed=from_packed)


def _dist():
    import torch.distributed as dist
    return dist


def _reduce_(arr, op: str, group=None):
    """In-place all-reduce of a numpy array or torch tensor (complex: as real
    pairs).  Device tensors stay on the device for NCCL; gloo works on host
    copies."""
    torch = _torch()
    dist = _dist()
    rop = dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM
    backend = dist.get_backend(group)
    if isinstance(arr, torch.Tensor):
        if arr.is_cuda and backend != "nccl":
            host = arr.cpu()
            dist.all_reduce(torch.view_as_real(host) if host.is_complex() else host, op=rop, group=group)
            arr.copy_(host)
            return arr
        dist.all_reduce(torch.view_as_real(arr) if arr.is_complex() else arr, op=rop, group=group)
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


def partition_model(B: int, world: int, hbm_gbs: float = 6540.0, link_gbs: float = 700.0,
                    compact_k1: bool = False) -> dict:
    """Per-adjoint time model (ms) of the two partitions for one rank at
    `world` ranks, excluding the window stage (the same in both): FFT passes
    at the HBM rate (3 passes x read + write x 16 B per cell; the single-GPU
    FFT is pruned to 2/3 of that), the basal adjoint (~0.5 ms at B = 64,
    x16 per doubling of B), the collectives at the NVLink bus rate."""
    n0, n1, n2 = 8 * B, (4 if compact_k1 else 8) * B, 4 * B
    pad = 16
    cells, padded = n0 * n1 * n2, n0 * (n1 + 2 * pad) * (n2 + 2 * pad)
    full_fft = 3 * 2 * 16.0 * cells / (hbm_gbs * 1e9) * 1e3
    basal = 0.5 * (B / 64.0) ** 4
    count = B * (B + 1) * (2 * B + 1) // 6
    coeffs = (2.0 / 3.0) * full_fft + basal + (2 * (world - 1) / world * 16.0 * count / (link_gbs * 1e9) * 1e3
                                              if world > 1 else 0.0)
    if world == 1:
        return {"coeffs": coeffs, "grid": coeffs, "choice": "coeffs"}
    rs = (world - 1) / world * 16.0 * padded / (link_gbs * 1e9) * 1e3
    slab2d = (2.0 / 3.0) * full_fft / world          # 2-D FFT of every plane, split over the ranks
    packed = n0 * (n1 // 2) * (2 * B) * 16.0
    gather = (world - 1) / world * packed / (link_gbs * 1e9) * 1e3
    root1d = 2 * 16.0 * padded / (hbm_gbs * 1e9) * 1e3 + basal
    grid = rs + slab2d + gather + root1d
    return {"coeffs": coeffs, "grid": grid, "choice": "coeffs" if coeffs <= grid else "grid"}


class ShardedPlan:
    """This rank's plan over its node shard; `adjoint` returns the global
    coefficient vector (identical on every rank)."""

    def __init__(self, B: int, local_points, *, group=None, rho: float | None = None,
                 compute: Compute | None = None, partition: str = "auto", **plan_kw):
        if partition not in ("auto", "coeffs", "grid"):
            raise ValueError("partition must be 'auto', 'coeffs' or 'grid'")
        dist = _dist()
        self.group = group
        self.B = int(B)
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.compute = compute or cuda_compute()
        self.rho = float(rho) if rho is not None else global_rho(local_points, group)
        self.plan = self.compute.plan(B, local_points, rho=self.rho, **plan_kw)
        if partition == "auto":
            partition = partition_model(B, self.world, compact_k1=bool(plan_kw.get("compact_k1")))["choice"]
        if partition == "grid" and self.compute.spread is None:
            raise ValueError("the grid partition needs the compute's stage functions")
        self.partition = partition

    def forward(self, coeffs):
        """Values at this rank's nodes (no collective)."""
        return self.compute.forward(self.plan, coeffs)

    def adjoint(self, local_values):
        """Sum over all ranks of the shard adjoints."""
        if self.partition == "coeffs" or self.world == 1:
            return _reduce_(self.compute.adjoint(self.plan, local_values), "sum", self.group)
        return self._adjoint_grid(local_values)

    def slab(self, n0: int) -> tuple[int, int]:
        """This rank's axis-0 planes [a0, a1) of the reduce-scatter."""
        return shard_bounds(n0, self.rank, self.world)

    def _adjoint_grid(self, local_values):
        torch = _torch()
        dist = _dist()
        c = self.compute
        host_in = not type(local_values).__module__.startswith("torch")
        grid = c.spread(self.plan, local_values)
        grid_t = grid if isinstance(grid, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(grid))
        n0, crop1, crop2 = c.grid_info(self.plan)
        a0, a1 = self.slab(n0)
        flat = grid_t.reshape(n0, -1)
        backend = dist.get_backend(self.group)
        # reduce-scatter of axis-0 plane blocks: rank k keeps planes [a0, a1), summed
        if backend == "nccl" and n0 % self.world == 0:
            out = flat[a0:a1]   # in place: NCCL allows recvbuff == sendbuff + rank * recvcount
            dist.reduce_scatter_tensor(torch.view_as_real(out), torch.view_as_real(flat), group=self.group)
        else:   # gloo / uneven blocks: all-reduce, keep the own block
            tmp = flat.cpu() if flat.is_cuda and backend != "nccl" else flat
            dist.all_reduce(torch.view_as_real(tmp), group=self.group)
            if tmp is not flat:
                flat[a0:a1].copy_(tmp[a0:a1])
        if not isinstance(grid, torch.Tensor):
            grid = grid_t.numpy()
        packed = c.slab_fft(self.plan, grid, a0, a1)
        packed_t = packed if isinstance(packed, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(packed))
        # gather of the packed planes to rank 0 (blocks padded to the largest
        # block when N0 does not divide evenly: gather needs equal sizes)
        use_host = packed_t.is_cuda and backend != "nccl"
        blk = -(-n0 // self.world)
        send = packed_t.cpu() if use_host else packed_t.contiguous()
        if send.shape[0] != blk:
            pad_ = torch.zeros((blk, crop1, crop2), dtype=send.dtype, device=send.device)
            pad_[:send.shape[0]] = send
            send = pad_
        if self.rank == 0:
            recv = torch.empty((self.world * blk, crop1, crop2), dtype=torch.complex128, device=send.device)
            dist.gather(torch.view_as_real(send), [torch.view_as_real(recv[k * blk:(k + 1) * blk])
                                                   for k in range(self.world)], dst=0, group=self.group)
            if blk * self.world == n0:
                full = recv
            else:
                full = torch.empty((n0, crop1, crop2), dtype=torch.complex128, device=send.device)
                for k in range(self.world):
                    b0, b1 = shard_bounds(n0, k, self.world)
                    full[b0:b1] = recv[k * blk:k * blk + (b1 - b0)]
        else:
            dist.gather(torch.view_as_real(send), None, dst=0, group=self.group)
        count = self.B * (self.B + 1) * (2 * self.B + 1) // 6
        if self.rank == 0:
            src = full.to(packed_t.device) if use_host else full
            coeffs = c.from_packed(self.plan, src if isinstance(packed, torch.Tensor) else src.numpy())
            coeffs = coeffs if isinstance(coeffs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(coeffs))
        else:
            coeffs = torch.empty((count,), dtype=torch.complex128, device=packed_t.device)
        if coeffs.is_cuda and backend != "nccl":
            h = coeffs.cpu()
            dist.broadcast(torch.view_as_real(h), src=0, group=self.group)
            coeffs.copy_(h)
        else:
            dist.broadcast(torch.view_as_real(coeffs), src=0, group=self.group)
        if host_in:
            return coeffs.cpu().numpy()
        return coeffs
