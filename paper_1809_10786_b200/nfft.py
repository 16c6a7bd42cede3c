"""The reference's NFFT layer (`sglnufft.nfft`, nfft.py:1-273) on the device.

Non-equispaced FFTs on the torus in d <= 3 dimensions,

    p(t) = sum_{k in I_n} w_k e^{+i <k, t>},   c_k = sum_i v_i e^{-i <k, t_i>},

with the same plan / execute / adjoint surface, centred coefficient layout
(position p on axis j holds frequency p - n_j/2), node reduction into
[0, 2 pi), oversampled lengths pow2(sigma n_j), Gaussian window and
ValueError conditions.  The work runs in `libsgl_b200.so` (the window
kernels, halo grid and cuFFT plan of the SGL transform, without its basal
stage): `sgl_nfft_plan_create` + `sgl_forward` / `sgl_adjoint`.

`ndft` / `ndft_adjoint` are the exact sums on the device (an exact plan).
`nfft_error_bound` is the reference's closed-form bound (host arithmetic).
d = 3 runs the tiled DMMA window kernels; d = 1, 2 are embedded as length-1
leading axes with a single unit-weight tap (exact, no window on them) and run
the per-node kernels.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .transform import _is_torch, _stream_ptr, _torch

_BACKENDS = ("auto", "tiled", "generic", "i8", "numba", "numpy")


def _as_axes(value, d: int, name: str) -> tuple:
    if np.ndim(value) == 0:
        return (int(value),) * d
    out = tuple(int(v) for v in value)
    if len(out) != d:
        raise ValueError(f"{name} must be scalar or length-{d}")
    return out


def _check_d(d: int) -> None:
    if d < 1 or d > 3:
        raise ValueError("only d <= 3 supported")


@dataclass
class NfftPlan:
    """Device plan mirroring the reference NfftPlan fields (nfft.py:101-120)."""
    d: int
    n_axis: tuple
    sigma: tuple
    q: int
    grid_shape: tuple
    sigma_eff: tuple
    lam: tuple
    nodes: object
    backend: str
    exact: bool = False
    _handle: int = field(default=0, repr=False)

    @property
    def m(self) -> int:
        return int(np.shape(self.nodes)[0])

    @property
    def deconv(self):
        """Per-axis 1/phi-hat over the centred range (nfft.py:183-186)."""
        return [np.exp(2 * self.lam[j] * (np.pi * (np.arange(n) - n // 2) / self.grid_shape[j]) ** 2)
                for j, n in enumerate(self.n_axis)]

    @property
    def guard(self) -> dict:
        """Accuracy-guard diagnostics of the int8 gather (backend="i8")."""
        i = _native.PlanInfo()
        _native.check(_native.lib().sgl_plan_get_info(self._handle, ctypes.byref(i)))
        return {"on": bool(i.guard), "fwd_fallbacks": int(i.guard_fwd_fallbacks),
                "adj_fallbacks": int(i.guard_adj_fallbacks), "est_fwd": float(i.guard_est_fwd),
                "est_adj": float(i.guard_est_adj)}

    def close(self) -> None:
        if self._handle:
            _native.lib().sgl_plan_destroy(self._handle)
            self._handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nfft_plan(d: int, n_axis, sigma, q: int, nodes, precompute: bool = True, backend: str = "auto",
              exact: bool = False) -> NfftPlan:
    """Plan the fast transform pair for one node set (nfft.py:147-207).

    ``nodes`` (m, d), reduced into [0, 2 pi).  ``sigma``: integer >= 2, or
    one per axis.  ``backend``:
    "auto" / "tiled" (FP64 DMMA kernels for d = 3, q <= 16; the int8 gather
    of SGL plans is not used here: a white NFFT spectrum amplifies its
    digit-split error to ~1e-10), "generic" (per-node kernels), "i8" (the int8
    gather, kept correct by the accuracy guard: a call whose error estimate
    exceeds 1e-11 is recomputed on the FP64 gather); the reference
    names "numba" / "numpy" are accepted as "auto".  ``precompute`` is accepted; windows are evaluated
    on the fly on the device.  ``exact=True`` plans the direct NDFT."""
    _check_d(d)
    n_axis = _as_axes(n_axis, d, "n_axis")
    sig = _as_axes(sigma, d, "sigma")
    if any(n < 2 or n % 2 for n in n_axis):
        raise ValueError("per-axis degree must be even and >= 2")
    if any(s < 2 for s in sig):
        raise ValueError("oversampling factor must be an integer >= 2")
    if q < 1:
        raise ValueError("cutoff parameter must be >= 1")
    if backend not in _BACKENDS:
        raise ValueError("backend must be 'auto', 'numba' or 'numpy'")
    grid = tuple(1 << int(np.ceil(np.log2(s * n))) for s, n in zip(sig, n_axis))
    if not exact and any(q >= g for g in grid):
        raise ValueError(f"cutoff q = {q} must be below sigma*n = {min(grid)}")
    torch_in = _is_torch(nodes)
    if torch_in:
        torch = _torch()
        pts = nodes.to(torch.float64).contiguous()
        if pts.dim() != 2 or pts.shape[1] != d:
            raise ValueError("nodes must be (m, d)")
        ptr, M = pts.data_ptr(), int(pts.shape[0])
    else:
        pts = np.ascontiguousarray(np.atleast_2d(np.asarray(nodes, dtype=np.float64)))
        if pts.ndim != 2 or pts.shape[1] != d:
            raise ValueError("nodes must be (m, d)")
        ptr, M = pts.ctypes.data, int(pts.shape[0])
    flags = 0
    if exact:
        flags |= _native.FLAG_EXACT_LAST_STAGE
    if backend == "generic":
        flags |= _native.FLAG_GENERIC_GRIDDING
    if backend == "i8":
        flags |= _native.FLAG_I8_GATHER
    n_arr = (ctypes.c_int32 * d)(*n_axis)
    s_arr = (ctypes.c_int32 * d)(*sig)
    h = ctypes.c_void_p(0)
    _native.check(_native.lib().sgl_nfft_plan_create(int(d), n_arr, M, ptr if M else None, s_arr, int(q), flags,
                                                     _stream_ptr(pts), ctypes.byref(h)))
    info = _native.PlanInfo()
    _native.check(_native.lib().sgl_plan_get_info(h, ctypes.byref(info)))
    return NfftPlan(d=d, n_axis=n_axis, sigma=sig, q=int(q), grid_shape=tuple(info.grid)[3 - d:],
                    sigma_eff=tuple(info.sigma_eff)[3 - d:], lam=tuple(info.lam)[3 - d:], nodes=pts,
                    backend="generic" if info.generic else ("i8" if info.i8_gather else "tiled"), exact=bool(exact),
                    _handle=h.value)


def nfft_execute(plan: NfftPlan, coeffs):
    """Approximate p(t_i) for coefficients on I_n (centred layout) (nfft.py:234-251)."""
    L = _native.lib()
    if _is_torch(coeffs):
        torch = _torch()
        c = coeffs.to(torch.complex128).contiguous()
        if tuple(c.shape) != plan.n_axis:
            raise ValueError(f"coefficient shape {tuple(c.shape)} != {plan.n_axis}")
        out = torch.empty((plan.m,), dtype=torch.complex128, device=c.device)
        _native.check(L.sgl_forward(plan._handle, c.data_ptr(), 1, out.data_ptr() if plan.m else None,
                                    _stream_ptr(c)))
        return out
    c = np.ascontiguousarray(coeffs, dtype=np.complex128)
    if c.shape != plan.n_axis:
        raise ValueError(f"coefficient shape {c.shape} != {plan.n_axis}")
    out = np.empty(plan.m, dtype=np.complex128)
    _native.check(L.sgl_forward(plan._handle, c.ctypes.data, 1, out.ctypes.data if plan.m else None, None))
    return out


def nfft_adjoint_execute(plan: NfftPlan, values):
    """Approximate adjoint sums c_k = sum_i v_i e^{-i<k,t_i>} (nfft.py:254-273)."""
    L = _native.lib()
    if _is_torch(values):
        torch = _torch()
        v = values.to(torch.complex128).contiguous()
        if tuple(v.shape) != (plan.m,):
            raise ValueError("values length must match the plan's node count")
        out = torch.empty(plan.n_axis, dtype=torch.complex128, device=v.device)
        _native.check(L.sgl_adjoint(plan._handle, v.data_ptr() if plan.m else None, out.data_ptr(),
                                    _stream_ptr(v)))
        return out
    v = np.ascontiguousarray(values, dtype=np.complex128)
    if v.shape != (plan.m,):
        raise ValueError("values length must match the plan's node count")
    out = np.empty(plan.n_axis, dtype=np.complex128)
    _native.check(L.sgl_adjoint(plan._handle, v.ctypes.data if plan.m else None, out.ctypes.data, None))
    return out


def ndft(d: int, n_axis, coeffs, nodes):
    """Exact sums p(t_i) = sum_k coeffs_k e^{i<k,t_i>} on the device (nfft.py:51-66)."""
    _check_d(d)
    n_axis = _as_axes(n_axis, d, "n_axis")
    if tuple(np.shape(coeffs)) != n_axis:
        raise ValueError(f"coefficient shape {tuple(np.shape(coeffs))} != {n_axis}")
    p = nfft_plan(d, n_axis, 2, 1, nodes, exact=True)
    try:
        return nfft_execute(p, coeffs)
    finally:
        p.close()


def ndft_adjoint(d: int, n_axis, values, nodes):
    """Exact adjoint sums c_k = sum_i values_i e^{-i<k,t_i>} on the device (nfft.py:69-82)."""
    _check_d(d)
    n_axis = _as_axes(n_axis, d, "n_axis")
    p = nfft_plan(d, n_axis, 2, 1, nodes, exact=True)
    try:
        return nfft_adjoint_execute(p, values)
    finally:
        p.close()


def nfft_error_bound(d: int, sigma: float, q: int, l1_norm: float) -> float:
    """Worst-case max-abs error of the Gaussian-window fast transform
    (the reference's closed form, nfft.py:85-98); host arithmetic."""
    s = float(sigma)
    if s < (np.sqrt(d) + 1) / 2:
        raise ValueError("oversampling factor too small for the bound")
    alias = (2.0 ** d - 1.0) * (2.0 + 1.0 / (np.pi * q)) ** d
    trunc = (3.0 ** d - 1.0) / q ** (d / 2.0) * (
        np.sqrt((2 * s - 1) / (2 * s)) + np.sqrt(2 * s / (2 * s - 1)) / (2 * np.pi)) ** d
    decay = np.exp(-q * np.pi * (1.0 - (1.0 + d / (2 * s - 1)) / (2 * s)))
    return float(l1_norm * (alias + trunc) * decay)
