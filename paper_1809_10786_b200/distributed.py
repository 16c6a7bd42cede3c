"""Multi-GPU NFSGLFT: node shards over a torch.distributed group.

One process per GPU.  The reference has no multi-GPU code; the
partition follows BASELINE's north star:

* forward (pointwise in the nodes): each rank evaluates its own node shard;
  the oversampled grid is rebuilt per rank (basal stage + FFT, ~1.6 ms at
  B = 64), cheaper than moving the 1.07 GB grid.  No collective.
* adjoint (a sum over nodes), two partitions:
  - ``partition="grid"`` (the north star's): each rank spreads its shard into
    its own oversampled grid.  The ranks OR the axis-0 planes their windows
    touch (the warped radius lives in [0, pi], so about half of the planes
    plus q on each side; `plane_pieces`) and an NCCL reduce-scatter over
    those planes combines the grids, each rank keeping a block of planes.
    Each rank runs the 2-D FFT (axes 1-2) of its planes and packs the
    spectral box the basal stage reads (1/4.8 of a plane at B = 64).  Then
    (``exchange="alltoall"``, the default) an all-to-all re-partitions the
    packed box from planes to columns, each rank runs the 1-D FFT along axis
    0 of its columns with the crop and deconvolution, the cropped spectrum
    eta (4B x crop1 x crop2) is gathered to rank 0, which runs the basal
    adjoint and broadcasts the coefficients.  ``exchange="gather"`` sends
    the packed planes to rank 0 instead and runs the 1-D FFT there.
  - ``partition="coeffs"``: each rank runs the whole adjoint of its shard and
    the ranks all-reduce the coefficient vector (1.4 MB at B = 64, 11 MB at
    B = 128).  The FFT and basal adjoint are linear, so reducing after them is
    exact; the FFT is replicated instead of split.
  ``partition="auto"`` picks by the bytes/time model `partition_model`
  (DESIGN.md section 6): on NVSwitch the grid reduce-scatter (0.72 GB of
  touched planes at B = 64, 5.3 GB at B = 128) costs more than the replicated
  FFT it saves, so "auto" is "coeffs" for the BASELINE configurations.
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


def shard_indices(points, rank: int, world: int, mode: str = "radial") -> np.ndarray:
    """Caller indices of rank's node shard (ascending), count-balanced.

    "contiguous": [start, stop) of the caller order (`shard_bounds`): for
    unordered inputs a random subsample, 1/world of the node density.
    "radial": the rank-th of `world` equal-count shells in r.  The warped
    radius is grid axis 0 (transform.py:46-55), so a shell covers one band of
    axis-0 planes at the full node density: the int8 window tiles stay as
    full as on one GPU (config 3 at 8 ranks: `tools/shard_probe.py`), and a
    rank's spread touches only its band plus q planes.
    "theta": equal-count bands in the polar angle theta = grid axis 1: whole
    rows of the window tiles' pencils, every radius and azimuth, i.e. full
    node density and the global range of output magnitudes on every rank."""
    if mode not in ("contiguous", "radial", "theta"):
        raise ValueError("mode must be 'contiguous', 'radial' or 'theta'")
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    M = pts.shape[0]
    s0, s1 = shard_bounds(M, rank, world)
    if mode == "contiguous":
        return np.arange(s0, s1)
    order = np.argsort(pts[:, 0 if mode == "radial" else 1], kind="stable")
    if mode == "radial" or M == 0:
        return np.sort(order[s0:s1])
    # theta: equal shares of estimated work rather than of nodes.  Near the
    # poles the nodes spread over more window tiles per node (the bands are
    # wider in theta and sparser in the grid): weight 1 + 0.25 (1 - sin theta)
    # evens the ranks' times at config 3, N = 8 (tools/shard_probe.py)
    wgt = 1.0 + 0.25 * (1.0 - np.sin(pts[order, 1]))
    cum = np.cumsum(wgt)
    edges = np.searchsorted(cum, cum[-1] * np.arange(world + 1) / world, side="left")
    edges[0], edges[-1] = 0, M
    return np.sort(order[edges[rank]:edges[rank + 1]])


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
    # the all-to-all exchange: ``planes(plan) -> uint8 (N0,)`` (planes the
    # shard's windows touch), ``axis0(plan, cols (N0, nc), col0) -> eta
    # block (4B, nc)``, ``from_eta(plan, eta (4B, crop1, crop2)) -> coeffs``
    planes: Callable | None = None
    axis0: Callable | None = None
    from_eta: Callable | None = None


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

    def planes(p):
        gi = grid_info(p)
        mask = np.zeros(gi.N0, dtype=np.uint8)
        _native.check(_native.lib().sgl_plan_planes(p._handle, mask.ctypes.data))
        return mask

    def axis0(p, cols, col0):
        torch = _torch()
        dev = torch.device("cuda", p.device)
        cols = torch.as_tensor(cols, device=dev).to(torch.complex128).contiguous()
        nc = int(cols.shape[1])
        out = torch.empty((4 * p.B, nc), dtype=torch.complex128, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _native.check(_native.lib().sgl_adjoint_axis0(p._handle, cols.data_ptr() if nc else None, nc, int(col0),
                                                      out.data_ptr() if nc else None, st))
        return out

    def from_eta(p, eta):
        torch = _torch()
        dev = torch.device("cuda", p.device)
        eta = torch.as_tensor(eta, device=dev).to(torch.complex128).contiguous()
        out = torch.empty((p.count,), dtype=torch.complex128, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _native.check(_native.lib().sgl_adjoint_from_eta(p._handle, eta.data_ptr(), out.data_ptr(), st))
        return out

    return Compute(transform.plan, transform.forward, transform.adjoint, spread=spread,
                   grid_info=lambda p: (lambda g: (g.N0, g.crop1, g.crop2))(grid_info(p)),
                   slab_fft=slab_fft, from_packed=from_packed, planes=planes, axis0=axis0, from_eta=from_eta)


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


def plane_pieces(mask, world: int) -> list[tuple[int, int, int, int]]:
    """The reduce-scatter layout over the touched axis-0 planes.

    `mask` (N0,) marks the planes any rank's windows touch.  The touched set
    is covered by the shortest circular arc (the complement of the largest
    run of untouched planes), split at the wrap into at most two pieces
    [ps, pe).  Each piece is widened to `world` equal blocks of `blk` planes
    starting at `s` (kept inside [0, N0), growing into untouched planes) so
    the reduce-scatter can run in place on the grid.  Returns
    [(s, blk, ps, pe)]; rank k owns planes [s + k blk, s + (k+1) blk) clipped
    to [ps, pe), so every touched plane has exactly one owner.  When widened
    pieces would overlap, one piece covers all planes (blk = ceil(N0/world);
    NCCL then needs world | N0, else the all-reduce fallback runs)."""
    mask = np.asarray(mask).astype(bool)
    n0 = mask.size
    if not mask.any():
        return []
    whole = [(0, -(-n0 // world), 0, n0)]
    if mask.all():
        return whole
    # largest circular run of untouched planes
    t = np.flatnonzero(mask)
    gaps = np.diff(np.concatenate([t, [t[0] + n0]])) - 1   # untouched run after each touched plane
    j = int(np.argmax(gaps))
    start = int((t[j] + gaps[j] + 1) % n0)                 # first touched plane after the largest gap
    length = n0 - int(gaps[j])
    if start + length <= n0:
        raw = [(start, start + length)]
    else:
        raw = [(start, n0), (0, start + length - n0)]
    pieces = []
    for ps, pe in raw:
        blk = -(-(pe - ps) // world)
        span = blk * world
        if span > n0:
            return whole
        s0 = ps if ps + span <= n0 else n0 - span           # grow upward, or downward at the top
        pieces.append((s0, blk, ps, pe))
    if len(pieces) == 2:
        (sa, ba, _, _), (sb, bb, _, _) = pieces
        if max(sa, sb) < min(sa + ba * world, sb + bb * world):
            return whole
    return pieces


def owned_planes(pieces, rank: int, world: int) -> list[tuple[int, int]]:
    """Rank's plane ranges [a0, a1) under `plane_pieces` (possibly empty)."""
    out = []
    for s0, blk, ps, pe in pieces:
        a0, a1 = max(ps, s0 + rank * blk), min(pe, s0 + (rank + 1) * blk)
        if a1 > a0:
            out.append((a0, a1))
    return out


def partition_model(B: int, world: int, hbm_gbs: float = 6540.0, link_gbs: float = 700.0,
                    compact_k1: bool = False, q: int = 16) -> dict:
    """Per-adjoint time model (ms) of the two partitions for one rank at
    `world` ranks, excluding the window stage (the same in both): FFT passes
    at the HBM rate (3 passes x read + write x 16 B per cell; the single-GPU
    FFT is pruned to 2/3 of that), the basal adjoint (~0.5 ms at B = 64,
    x16 per doubling of B), the collectives at the NVLink bus rate.  The grid
    partition moves only the touched planes: the warped radius spans [0, pi],
    half of axis 0, plus q planes on either side."""
    n0, n1, n2 = 8 * B, (4 if compact_k1 else 8) * B, 4 * B
    pad = 16
    touched = min(n0, n0 // 2 + 2 * q + 1)
    cells = n0 * n1 * n2
    full_fft = 3 * 2 * 16.0 * cells / (hbm_gbs * 1e9) * 1e3
    basal = 0.5 * (B / 64.0) ** 4
    count = B * (B + 1) * (2 * B + 1) // 6
    coeffs = (2.0 / 3.0) * full_fft + basal + (2 * (world - 1) / world * 16.0 * count / (link_gbs * 1e9) * 1e3
                                              if world > 1 else 0.0)
    if world == 1:
        return {"coeffs": coeffs, "grid": coeffs, "choice": "coeffs"}
    plane = (n1 + 2 * pad) * (n2 + 2 * pad) * 16.0
    rs = (world - 1) / world * touched * plane / (link_gbs * 1e9) * 1e3
    slab2d = 2 * 2 * 16.0 * touched * n1 * n2 / world / (hbm_gbs * 1e9) * 1e3   # 2-D FFT of the own planes
    box = (n1 // 2) * (2 * B) * 16.0                     # packed spectral box per plane
    a2a = (world - 1) / world * touched * box / world / (link_gbs * 1e9) * 1e3
    fft1 = 2 * 16.0 * n0 * (n1 // 2) * (2 * B) / world / (hbm_gbs * 1e9) * 1e3
    eta = (world - 1) / world * 4 * B * (n1 // 2) * (2 * B) * 16.0 / (link_gbs * 1e9) * 1e3
    grid = rs + slab2d + a2a + fft1 + eta + basal
    return {"coeffs": coeffs, "grid": grid, "choice": "coeffs" if coeffs <= grid else "grid"}


class ShardedPlan:
    """This rank's plan over its node shard; `adjoint` returns the global
    coefficient vector (identical on every rank)."""

    def __init__(self, B: int, local_points, *, group=None, rho: float | None = None,
                 compute: Compute | None = None, partition: str = "auto", exchange: str = "alltoall",
                 **plan_kw):
        if partition not in ("auto", "coeffs", "grid"):
            raise ValueError("partition must be 'auto', 'coeffs' or 'grid'")
        if exchange not in ("alltoall", "gather"):
            raise ValueError("exchange must be 'alltoall' or 'gather'")
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
        if partition == "grid" and exchange == "alltoall" and self.compute.axis0 is None:
            raise ValueError("the all-to-all exchange needs the compute's planes/axis0/from_eta")
        self.partition = partition
        self.exchange = exchange
        self.last_pieces = None   # plane_pieces of the last grid adjoint (diagnostics)

    def forward(self, coeffs):
        """Values at this rank's nodes (no collective)."""
        return self.compute.forward(self.plan, coeffs)

    def adjoint(self, local_values):
        """Sum over all ranks of the shard adjoints."""
        if self.partition == "coeffs" or self.world == 1:
            return _reduce_(self.compute.adjoint(self.plan, local_values), "sum", self.group)
        return self._adjoint_grid(local_values)

    def _collective_host(self, t):
        """gloo works on host tensors: (tensor for the collective, copy-back flag)."""
        if t.is_cuda and _dist().get_backend(self.group) != "nccl":
            return t.cpu(), True
        return t, False

    def _reduce_planes(self, flat, pieces, n0):
        """Sum the ranks' grids over the pieces; this rank's owned planes end up
        reduced in `flat` (other planes are left partially summed)."""
        torch = _torch()
        dist = _dist()
        nccl = dist.get_backend(self.group) == "nccl"
        for s0, blk, ps, pe in pieces:
            span = blk * self.world
            region = flat[s0:s0 + span] if s0 + span <= n0 else flat[s0:]
            if nccl and region.shape[0] == span:
                out = region[self.rank * blk:(self.rank + 1) * blk]   # in place: recvbuff = sendbuff + rank * count
                dist.reduce_scatter_tensor(torch.view_as_real(out), torch.view_as_real(region), group=self.group)
            else:   # gloo / uneven: all-reduce the piece
                tmp, back = self._collective_host(region)
                dist.all_reduce(torch.view_as_real(tmp), group=self.group)
                if back:
                    region.copy_(tmp.to(region.device))

    def _adjoint_grid(self, local_values):
        torch = _torch()
        dist = _dist()
        c = self.compute
        host_in = not type(local_values).__module__.startswith("torch")
        grid = c.spread(self.plan, local_values)
        as_np = not isinstance(grid, torch.Tensor)
        grid_t = torch.from_numpy(np.ascontiguousarray(grid)) if as_np else grid
        n0, crop1, crop2 = c.grid_info(self.plan)
        flat = grid_t.reshape(n0, -1)
        # the planes any rank touches, and the reduce-scatter layout over them
        if c.planes is not None:
            mask = _reduce_(np.asarray(c.planes(self.plan)).astype(np.int32), "max", self.group)
            pieces = plane_pieces(mask, self.world)
        else:
            pieces = plane_pieces(np.ones(n0, dtype=bool), self.world)
        self.last_pieces = pieces
        self._reduce_planes(flat, pieces, n0)
        if as_np:
            grid = grid_t.numpy().reshape(np.shape(grid))
        owned = [owned_planes(pieces, k, self.world) for k in range(self.world)]
        parts = [c.slab_fft(self.plan, grid, a0, a1) for a0, a1 in owned[self.rank]]
        parts = [x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x)) for x in parts]
        dev = grid_t.device
        packed = (torch.cat(parts) if parts else
                  torch.zeros((0, crop1, crop2), dtype=torch.complex128, device=dev))
        if self.exchange == "alltoall":
            coeffs = self._finish_alltoall(packed, owned, n0, crop1, crop2, as_np)
        else:
            coeffs = self._finish_gather(packed, owned, n0, crop1, crop2, as_np)
        coeffs = coeffs if isinstance(coeffs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(coeffs))
        if coeffs.device != dev:
            coeffs = coeffs.to(dev)
        h, back = self._collective_host(coeffs)
        dist.broadcast(torch.view_as_real(h), src=0, group=self.group)
        if back:
            coeffs.copy_(h.to(dev))
        if host_in:
            return coeffs.cpu().numpy()
        return coeffs

    def _empty_coeffs(self, device):
        torch = _torch()
        count = self.B * (self.B + 1) * (2 * self.B + 1) // 6
        return torch.empty((count,), dtype=torch.complex128, device=device)

    def _finish_alltoall(self, packed, owned, n0, crop1, crop2, as_np):
        """planes -> columns all-to-all, 1-D FFT along axis 0 of the own
        columns (+ crop, deconvolution), eta gathered to rank 0, basal
        adjoint there.  Returns the coefficients on rank 0 (else a buffer)."""
        torch = _torch()
        dist = _dist()
        c = self.compute
        dev = packed.device
        C = crop1 * crop2
        cols = [shard_bounds(C, k, self.world) for k in range(self.world)]
        n_own = [sum(a1 - a0 for a0, a1 in o) for o in owned]
        P = packed.reshape(n_own[self.rank], C)
        send = torch.cat([P[:, c0:c1].reshape(-1) for c0, c1 in cols])
        mc0, mc1 = cols[self.rank]
        ncm = mc1 - mc0
        recv = torch.empty((sum(n_own) * ncm,), dtype=torch.complex128, device=dev)
        s_h, s_back = self._collective_host(send)
        r_h, r_back = self._collective_host(recv)
        dist.all_to_all_single(torch.view_as_real(r_h), torch.view_as_real(s_h),
                               output_split_sizes=[n * ncm for n in n_own],
                               input_split_sizes=[n_own[self.rank] * (c1 - c0) for c0, c1 in cols], group=self.group)
        if r_back:
            recv = r_h.to(dev)
        # the own columns of every plane (untouched planes are zero)
        X = torch.zeros((n0, ncm), dtype=torch.complex128, device=dev)
        off = 0
        for k in range(self.world):
            for a0, a1 in owned[k]:
                n = (a1 - a0) * ncm
                X[a0:a1] = recv[off:off + n].reshape(a1 - a0, ncm)
                off += n
        eta = c.axis0(self.plan, X.numpy() if as_np else X, mc0)
        eta = eta if isinstance(eta, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(eta))
        eta = eta.to(dev)
        # gather of the eta column blocks to rank 0 (padded to equal sizes)
        W = 4 * self.B
        mx = max(c1 - c0 for c0, c1 in cols)
        blk = torch.zeros((W, mx), dtype=torch.complex128, device=dev)
        blk[:, :ncm] = eta
        b_h, _ = self._collective_host(blk)
        if self.rank == 0:
            bufs = [torch.empty_like(b_h) for _ in range(self.world)]
            dist.gather(torch.view_as_real(b_h), [torch.view_as_real(b) for b in bufs], dst=0, group=self.group)
            full = torch.empty((W, C), dtype=torch.complex128, device=b_h.device)
            for k, (c0, c1) in enumerate(cols):
                full[:, c0:c1] = bufs[k][:, :c1 - c0]
            full = full.reshape(W, crop1, crop2)
            return c.from_eta(self.plan, full.numpy() if as_np else full.to(dev))
        dist.gather(torch.view_as_real(b_h), None, dst=0, group=self.group)
        return self._empty_coeffs(dev)

    def _finish_gather(self, packed, owned, n0, crop1, crop2, as_np):
        """The packed planes gathered to rank 0 (padded to equal sizes), which
        runs the 1-D FFT along axis 0, crop, deconvolution and basal adjoint."""
        torch = _torch()
        dist = _dist()
        c = self.compute
        dev = packed.device
        n_own = [sum(a1 - a0 for a0, a1 in o) for o in owned]
        mx = max(max(n_own), 1)
        send = torch.zeros((mx, crop1, crop2), dtype=torch.complex128, device=dev)
        send[:n_own[self.rank]] = packed
        s_h, _ = self._collective_host(send)
        if self.rank == 0:
            bufs = [torch.empty_like(s_h) for _ in range(self.world)]
            dist.gather(torch.view_as_real(s_h), [torch.view_as_real(b) for b in bufs], dst=0, group=self.group)
            full = torch.zeros((n0, crop1, crop2), dtype=torch.complex128, device=s_h.device)
            for k in range(self.world):
                off = 0
                for a0, a1 in owned[k]:
                    full[a0:a1] = bufs[k][off:off + a1 - a0]
                    off += a1 - a0
            return c.from_packed(self.plan, full.numpy() if as_np else full.to(dev))
        dist.gather(torch.view_as_real(s_h), None, dst=0, group=self.group)
        return self._empty_coeffs(dev)
