"""B200 drop-in for the reference `plan / forward / adjoint` (transform.py:320-429).

Same names, argument meaning and ValueError conditions as the reference
`sglnufft.transform`; the work runs in `libsgl_b200.so` (hand-written
sm_100a kernels + cuFFT) through the C ABI of `include/sgl_b200.h`.

Inputs may be numpy arrays (host; results come back as numpy) or CUDA
`torch` tensors (device; results stay on the device as torch tensors).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .generate import coeff_count

_BACKENDS = ("auto", "tiled", "generic", "i8", "numba", "numpy")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _torch():
    import torch
    return torch


@dataclass
class NfftInfo:
    """Geometry of the oversampled grid (mirrors NfftPlan fields, nfft.py:101-120)."""
    d: int
    n_axis: tuple
    sigma: tuple
    q: int
    grid_shape: tuple
    sigma_eff: tuple
    lam: tuple
    backend: str

    @property
    def deconv(self):
        """Per-axis 1/phi-hat over the centred range (nfft.py:183-186)."""
        return [np.exp(2 * self.lam[j] * (np.pi * (np.arange(n) - n // 2) / self.grid_shape[j]) ** 2)
                for j, n in enumerate(self.n_axis)]


@dataclass
class SglPlan:
    """Per-point-set plan; owns the device state of libsgl_b200 (sorted nodes,
    window tiles, basal matrices, cuFFT plan, scratch grid).

    Shareable across threads and streams like the reference's plan
    (README.md:66-67): the library serialises calls on one plan."""
    B: int
    rho: float
    sigma: int
    q: int | None
    exact: bool
    compact_k1: bool
    points: object
    n_axis: tuple
    nfft: NfftInfo | None
    device: int
    _handle: int = field(repr=False)
    _info: _native.PlanInfo = field(repr=False)
    backend: str = "auto"
    precise_tables: bool = False
    flags: int = 0
    _twin: object = field(default=None, repr=False)   # extended-precision twin for precise=True calls

    @property
    def m_points(self) -> int:
        return int(self._info.M)

    @property
    def count(self) -> int:
        return int(self._info.coeff_count)

    @property
    def nodes(self) -> np.ndarray:
        """Warped torus nodes (transform.py:46-55), computed on request."""
        pts = self.points.detach().cpu().numpy() if _is_torch(self.points) else np.asarray(self.points)
        out = np.array(pts, dtype=float)
        out[:, 0] = np.arccos(np.clip((2 * out[:, 0] - self.rho) / self.rho, -1.0, 1.0))
        return out

    @property
    def r_nodes(self) -> np.ndarray:
        """Radial Chebyshev nodes rho (1 + cos w_j) / 2, w_j = (2j+1) pi / 4B
        (transform.py:365); the device folds them into its radial matrices."""
        w = (2 * np.arange(2 * self.B) + 1) * np.pi / (4 * self.B)
        return self.rho * (1 + np.cos(w)) / 2

    @property
    def tiles(self) -> int:
        return int(self._info.n_tiles)

    @property
    def stats(self) -> dict:
        """Plan statistics; `i8_scatter` is the adjoint's current engine (an
        automatic int8 choice can switch itself off at run time)."""
        i = _native.PlanInfo()
        _native.check(_native.lib().sgl_plan_get_info(self._handle, ctypes.byref(i)))
        return {"n_tiles": int(i.n_tiles), "tile_nodes": int(i.tile_nodes), "tile_dmma": int(i.tile_dmma),
                "generic": bool(i.generic), "plan_ms": float(i.plan_ms), "i8_gather": bool(i.i8_gather),
                "i8_tiles": int(i.i8_tiles), "i8_ksteps": int(i.i8_ksteps), "i8_scatter": bool(i.i8_scatter),
                "i8_sksteps": int(i.i8_sksteps), "guard": bool(i.guard), "guard_ap": float(i.guard_ap)}

    @property
    def guard(self) -> dict:
        """Accuracy-guard diagnostics of the int8 engines (reads device state)."""
        i = _native.PlanInfo()
        _native.check(_native.lib().sgl_plan_get_info(self._handle, ctypes.byref(i)))
        return {"on": bool(i.guard), "fwd_fallbacks": int(i.guard_fwd_fallbacks),
                "adj_fallbacks": int(i.guard_adj_fallbacks), "est_fwd": float(i.guard_est_fwd),
                "est_adj": float(i.guard_est_adj), "adj_response": float(i.guard_ap)}

    def stage_ms(self, direction: str = "forward") -> dict:
        """Per-stage device ms of the last call (plan(..., profile=True))."""
        buf = (ctypes.c_float * 5)()
        _native.check(_native.lib().sgl_plan_stage_ms(self._handle, 0 if direction == "forward" else 1, buf, 5))
        return dict(zip(_native.STAGES, (float(x) for x in buf)))

    def close(self) -> None:
        if self._twin is not None:
            self._twin.close()
            self._twin = None
        if self._handle:
            _native.lib().sgl_plan_destroy(self._handle)
            self._handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream_ptr(x) -> int | None:
    if _is_torch(x) and x.is_cuda:
        return _torch().cuda.current_stream(x.device).cuda_stream
    return None


def plan(B: int, points, sigma: int = 2, q: int | None = 16, rho: float | None = None,
         exact_last_stage: bool = False, compact_k1: bool = False, backend: str = "auto",
         precompute: bool = True, device: int | None = None, profile: bool = False,
         precise_tables: bool | None = None, flags: int = 0, devices=None,
         deterministic: bool = False) -> SglPlan:
    """Prepare a fast-transform plan for one scattered point set (transform.py:320-382).

    ``backend``: "auto" (q <= 16: the int8 tensor-core gather for the
    forward window stage (FP64 results by digit split) and the tiled FP64 DMMA
    scatter; per-node kernels otherwise), "tiled" (FP64 DMMA kernels in both
    directions), "generic" (per-node kernels), "i8" (int8 tensor-core engines
    in both directions for any node set; "auto" takes the int8 scatter only for
    large dense node sets).  Every int8 call is covered by the accuracy guard
    (csrc/guard.cu): a call whose digit-split error estimate exceeds 1e-11, or
    whose input is not finite, is recomputed on the FP64 kernels.  ``flags``
    adds raw `SGL_FLAG_*` bits of the C ABI (experiments).  The reference names
    "numba" / "numpy" are accepted as aliases of "auto".  ``precompute`` is
    accepted for compatibility: window weights are always evaluated on the
    fly on the device.  ``exact_last_stage=True`` replaces the window
    evaluation by the direct NDFT on the device (O(M n^3): verification).
    ``devices``: a list of CUDA device ids -- one plan over all of them in
    this process (node shards, one sub-plan per device, sgl_plan_create_multi);
    the one-process-per-GPU path is `distributed.ShardedPlan`.
    ``deterministic=True``: bitwise reproducible adjoints (the reference's
    serial spreading loop, _gridding.py:77-95, is): every window kernel reduces
    64-bit fixed-point integers into the grid instead of FP64 atomics
    (SGL_FLAG_DETERMINISTIC, csrc/determ.cu); costs one plan-time spread and a
    grid conversion per adjoint."""
    if B < 1:
        raise ValueError("bandwidth must be >= 1")
    if backend not in _BACKENDS:
        raise ValueError("backend must be 'auto', 'tiled', 'generic', 'i8', 'numba' or 'numpy'")
    torch_in = _is_torch(points)
    if torch_in:
        torch = _torch()
        pts = points.to(torch.float64)
        if pts.dim() == 1:
            pts = pts.reshape(1, -1)
        if pts.dim() != 2 or pts.shape[1] != 3:
            raise ValueError("points must be (M, 3) spherical coordinates")
        pts = pts.contiguous()
        ptr, M = pts.data_ptr(), int(pts.shape[0])
        dev = pts.device.index if pts.is_cuda else device
    else:
        pts = np.atleast_2d(np.ascontiguousarray(points, dtype=np.float64))
        if pts.ndim != 2 or pts.shape[1] != 3:
            raise ValueError("points must be (M, 3) spherical coordinates")
        ptr, M = pts.ctypes.data, int(pts.shape[0])
        dev = device
    if rho is not None and not rho > 0:
        raise ValueError("rho must be positive")
    if not exact_last_stage:   # window parameters only matter for the fast path (transform.py:352-356)
        if q is None or q < 1:
            raise ValueError("cutoff parameter q must be >= 1")
        if q >= 4 * sigma * B:
            raise ValueError(f"cutoff q = {q} must be below 4*sigma*B = {4 * sigma * B}")
        if backend == "tiled" and q > 16:
            raise ValueError("tiled window kernels need q <= 16")
    L = _native.lib()
    if dev is not None:
        _native.check(L.sgl_set_device(int(dev)))
    flags = int(flags)
    if backend == "i8":
        flags |= _native.FLAG_I8_SCATTER
    if exact_last_stage:
        flags |= _native.FLAG_EXACT_LAST_STAGE
    if compact_k1:
        flags |= _native.FLAG_COMPACT_K1
    if backend == "generic":
        flags |= _native.FLAG_GENERIC_GRIDDING
    if backend == "tiled":
        flags |= _native.FLAG_FP64_WINDOW
    if profile:
        flags |= _native.FLAG_PROFILE
    if deterministic:
        flags |= _native.FLAG_DETERMINISTIC
    # basal matrices in x87 extended precision by default (closer to the
    # truth on ill-conditioned configurations; SGL_FLAG_FP64_TABLES opts out)
    if precise_tables is None:
        precise_tables = not (flags & _native.FLAG_FP64_TABLES)
    if precise_tables:
        flags |= _native.FLAG_PRECISE
    else:
        flags |= _native.FLAG_FP64_TABLES
    h = ctypes.c_void_p(0)
    stream = _stream_ptr(pts)
    if devices is not None and len(devices) > 1:
        devs = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
        _native.check(L.sgl_plan_create_multi(int(B), M, ptr if M else None, int(sigma), int(q or 0),
                                              float(rho) if rho is not None else 0.0, flags, len(devices), devs,
                                              ctypes.byref(h)))
        dev = int(devices[0])
    else:
        if devices is not None and len(devices) == 1:
            dev = int(devices[0])
            _native.check(L.sgl_set_device(dev))
        _native.check(L.sgl_plan_create(int(B), M, ptr if M else None, int(sigma), int(q or 0),
                                        float(rho) if rho is not None else 0.0, flags, stream, ctypes.byref(h)))
    info = _native.PlanInfo()
    _native.check(L.sgl_plan_get_info(h, ctypes.byref(info)))
    nf = None if exact_last_stage else NfftInfo(
        3, tuple(info.n_axis), tuple(info.sigma_axes), int(q), tuple(info.grid), tuple(info.sigma_eff),
        tuple(info.lam), "generic" if info.generic else ("i8" if info.i8_gather else "tiled"))
    return SglPlan(B=int(B), rho=float(info.rho), sigma=int(sigma), q=None if exact_last_stage else int(q),
                   exact=bool(exact_last_stage),
                   compact_k1=bool(compact_k1), points=points, n_axis=tuple(info.n_axis), nfft=nf,
                   device=int(dev) if dev is not None else 0, _handle=h.value, _info=info, backend=backend,
                   precise_tables=bool(precise_tables), flags=int(flags))


def _for_call(p: SglPlan, precise: bool) -> SglPlan:
    """precise=True (the reference's 80-bit recurrences, recurrences.py:13):
    run on a twin plan whose basal tables were built in x87 extended
    precision (built on first use, cached on the plan)."""
    if not precise or p.precise_tables:
        return p
    if p._twin is None:
        p._twin = plan(p.B, p.points, sigma=p.sigma, q=p.q if not p.exact else 16, rho=p.rho,
                       exact_last_stage=p.exact, compact_k1=p.compact_k1, backend=p.backend, device=p.device,
                       precise_tables=True, flags=p.flags)
    return p._twin


def forward(p: SglPlan, coeffs, precise: bool = False):
    """Evaluate the expansion at the plan's points (transform.py:385-395).

    ``coeffs``: (count,) complex128, or (K, count) for K vectors on one plan
    (the batched forward).  Returns (M,) or (K, M)."""
    p = _for_call(p, precise)
    cnt = p.count
    if _is_torch(coeffs):
        torch = _torch()
        c = coeffs.to(torch.complex128).contiguous()
        if c.shape[-1:] != (cnt,) or c.dim() > 2:
            raise ValueError("coefficient length does not match the bandwidth")
        K = 1 if c.dim() == 1 else int(c.shape[0])
        out = torch.empty((K, p.m_points) if c.dim() == 2 else (p.m_points,), dtype=torch.complex128,
                          device=c.device)
        _native.check(_native.lib().sgl_forward(p._handle, c.data_ptr(), K, out.data_ptr() if out.numel() else None,
                                                _stream_ptr(c)))
        return out
    c = np.ascontiguousarray(coeffs, dtype=np.complex128)
    if c.shape[-1:] != (cnt,) or c.ndim > 2 or c.ndim == 0:
        raise ValueError("coefficient length does not match the bandwidth")
    K = 1 if c.ndim == 1 else c.shape[0]
    out = np.empty((K, p.m_points) if c.ndim == 2 else (p.m_points,), dtype=np.complex128)
    _native.check(_native.lib().sgl_forward(p._handle, c.ctypes.data, K, out.ctypes.data if out.size else None,
                                            None))
    return out


def adjoint(p: SglPlan, values, precise: bool = False):
    """Apply the conjugate transpose of `forward` (transform.py:398-429)."""
    p = _for_call(p, precise)
    if _is_torch(values):
        torch = _torch()
        v = values.to(torch.complex128).contiguous()
        if tuple(v.shape) != (p.m_points,):
            raise ValueError("values length does not match the plan")
        out = torch.empty((p.count,), dtype=torch.complex128, device=v.device)
        _native.check(_native.lib().sgl_adjoint(p._handle, v.data_ptr() if v.numel() else None, out.data_ptr(),
                                                _stream_ptr(v)))
        return out
    v = np.ascontiguousarray(values, dtype=np.complex128)
    if v.shape != (p.m_points,):
        raise ValueError("values length does not match the plan")
    out = np.empty(p.count, dtype=np.complex128)
    _native.check(_native.lib().sgl_adjoint(p._handle, v.ctypes.data if v.size else None, out.ctypes.data, None))
    return out


def forward_adjoint(p: SglPlan, coeffs, values):
    """``(forward(p, coeffs), adjoint(p, values))`` in one library call.

    The two inputs are independent; with host (numpy) arrays the library
    overlaps the value upload with the forward and the value download with
    the adjoint (sgl_forward_adjoint): fully asynchronously for page-locked
    arrays (e.g. ``torch.empty(..., pin_memory=True).numpy()``); for ordinary
    pageable arrays each copy is issued after the kernels it overlaps are
    enqueued (the copy call blocks the host, the GPU keeps computing).  Same
    checks as `forward`/`adjoint`."""
    cnt, M = p.count, p.m_points
    L = _native.lib()
    if _is_torch(coeffs) or _is_torch(values):
        torch = _torch()
        c = torch.as_tensor(coeffs).to(torch.complex128).contiguous()
        v = torch.as_tensor(values).to(torch.complex128).contiguous()
        if tuple(c.shape) != (cnt,):
            raise ValueError("coefficient length does not match the bandwidth")
        if tuple(v.shape) != (M,):
            raise ValueError("values length does not match the plan")
        dev = c.device if c.is_cuda else v.device
        out_v = torch.empty((M,), dtype=torch.complex128, device=dev)
        out_c = torch.empty((cnt,), dtype=torch.complex128, device=dev)
        _native.check(L.sgl_forward_adjoint(p._handle, c.data_ptr(), out_v.data_ptr() if M else None,
                                            v.data_ptr() if M else None, out_c.data_ptr(),
                                            _stream_ptr(out_c)))
        return out_v, out_c
    c = np.ascontiguousarray(coeffs, dtype=np.complex128)
    v = np.ascontiguousarray(values, dtype=np.complex128)
    if c.shape != (cnt,):
        raise ValueError("coefficient length does not match the bandwidth")
    if v.shape != (M,):
        raise ValueError("values length does not match the plan")
    out_v = np.empty(M, dtype=np.complex128)
    out_c = np.empty(cnt, dtype=np.complex128)
    _native.check(L.sgl_forward_adjoint(p._handle, c.ctypes.data, out_v.ctypes.data if M else None,
                                        v.ctypes.data if M else None, out_c.ctypes.data, None))
    return out_v, out_c


def _direct_points(points):
    if _is_torch(points):
        torch = _torch()
        pts = points.to(torch.float64)
        pts = (pts.reshape(1, -1) if pts.dim() == 1 else pts).contiguous()
        if pts.dim() != 2 or pts.shape[1] != 3:
            raise ValueError("points must be (M, 3) spherical coordinates")
        return pts, pts.data_ptr(), int(pts.shape[0])
    pts = np.atleast_2d(np.ascontiguousarray(points, dtype=np.float64))
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValueError("points must be (M, 3) spherical coordinates")
    return pts, pts.ctypes.data, int(pts.shape[0])


def evaluate_direct(coeffs, B: int, points):
    """Direct summation of the expansion at the points, on the device
    (reference transform.py:95-117; O(M * count): verification / the CLI's
    ``--method naive``)."""
    if B < 1:
        raise ValueError("bandwidth must be >= 1")
    pts, pptr, M = _direct_points(points)
    cnt = coeff_count(B)
    L = _native.lib()
    if _is_torch(coeffs) or _is_torch(points):
        torch = _torch()
        dev = next(x.device for x in (coeffs, points) if _is_torch(x))
        c = torch.as_tensor(coeffs, device=dev).to(torch.complex128).contiguous()
        if tuple(c.shape) != (cnt,):
            raise ValueError("coefficient length does not match the bandwidth")
        pts = torch.as_tensor(pts, device=c.device)
        out = torch.empty((M,), dtype=torch.complex128, device=c.device)
        _native.check(L.sgl_direct_forward(int(B), M, pts.data_ptr() if M else None, c.data_ptr(),
                                           out.data_ptr() if M else None, _stream_ptr(out)))
        return out
    c = np.ascontiguousarray(coeffs, dtype=np.complex128)
    if c.shape != (cnt,):
        raise ValueError("coefficient length does not match the bandwidth")
    out = np.empty(M, dtype=np.complex128)
    _native.check(L.sgl_direct_forward(int(B), M, pptr if M else None, c.ctypes.data,
                                       out.ctypes.data if M else None, None))
    return out


def evaluate_direct_adjoint(values, B: int, points):
    """Direct adjoint sums c_mu = sum_i v_i conj(H_mu(x_i)) on the device
    (reference transform.py:120-139)."""
    if B < 1:
        raise ValueError("bandwidth must be >= 1")
    pts, pptr, M = _direct_points(points)
    cnt = coeff_count(B)
    L = _native.lib()
    if _is_torch(values) or _is_torch(points):
        torch = _torch()
        dev = next(x.device for x in (values, points) if _is_torch(x))
        v = torch.as_tensor(values, device=dev).to(torch.complex128).contiguous()
        if tuple(v.shape) != (M,):
            raise ValueError("values length does not match the point count")
        pts = torch.as_tensor(pts, device=v.device)
        out = torch.empty((cnt,), dtype=torch.complex128, device=v.device)
        _native.check(L.sgl_direct_adjoint(int(B), M, pts.data_ptr() if M else None,
                                           v.data_ptr() if M else None, out.data_ptr(), _stream_ptr(out)))
        return out
    v = np.ascontiguousarray(values, dtype=np.complex128)
    if v.shape != (M,):
        raise ValueError("values length does not match the point count")
    out = np.empty(cnt, dtype=np.complex128)
    _native.check(L.sgl_direct_adjoint(int(B), M, pptr if M else None, v.ctypes.data if M else None,
                                       out.ctypes.data, None))
    return out


def transform_points(points, rho: float) -> np.ndarray:
    """Warp (r, theta, phi) to torus nodes (arccos((2r - rho)/rho), theta, phi)
    (reference transform.py:46-55; host arithmetic, the device warps its own
    copy in `plan`)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    r = pts[:, 0]
    if np.any(r > rho * (1 + 1e-12)):
        raise ValueError("point radius exceeds the radial parameter rho")
    out = pts.copy()
    out[:, 0] = np.arccos(np.clip((2 * r - rho) / rho, -1.0, 1.0))
    return out


def sgl_basis_eval(idx, point):
    """One basis function H_{n,l,m} at (r, theta, phi) points (reference
    special.py:171-182), by the device direct sum with a unit coefficient."""
    from .indexing import nlm_to_mu
    n, l, m = (int(v) for v in idx)
    mu = nlm_to_mu(n, l, m)
    p = np.asarray(point, dtype=float)
    shape = p.shape[:-1]
    c = np.zeros(coeff_count(n), dtype=np.complex128)
    c[mu] = 1.0
    out = evaluate_direct(c, n, p.reshape(-1, 3)).reshape(shape)
    return out if out.ndim else complex(out)


def growth_threshold(rho: float) -> float:
    """Bandwidth below which the small-radius branch of `error_bound` applies
    (the reference's closed form, transform.py:436-443)."""
    if not 0 < rho < 1:
        raise ValueError("threshold is defined for 0 < rho < 1")
    ie = 1.0 / np.e
    return float((np.exp(2 * ie) * (rho ** (2 * ie) - 1) / (2 * np.log(rho))) ** (1 - ie) - 0.5)


def error_bound(B: int, rho: float, q: int, l1_norm: float) -> float:
    """Analytic envelope of the fast path's max-abs error with unit leading
    constant (the reference's certificate, transform.py:446-462): a trend
    check in q, rho and B, not an acceptance threshold.  Host arithmetic."""
    ie = 1.0 / np.e
    small = rho < 1 and B <= growth_threshold(rho)
    a = 1.0 if small else 1.0 / rho
    b = 0.5 * np.exp(2 * ie) * (1.0 if small else rho ** (2 * ie))
    return float(B ** 3.5 * a * np.exp(b * (B + 0.5) ** (1 - ie) + 0.5 * rho ** 2 - 0.5 * np.pi * q) * l1_norm)


def choose_rho(points) -> float:
    """Largest sample radius; 1.0 if all points sit at the origin (transform.py:39-43)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    r = float(np.max(pts[:, 0])) if pts.size else 0.0
    return r if r > 0 else 1.0
