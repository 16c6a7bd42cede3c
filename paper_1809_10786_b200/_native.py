"""ctypes binding of the in-tree C ABI (`include/sgl_b200.h`).

There is no CPU fallback: if `_lib/libsgl_b200.so` is missing or fails to
load, every entry point raises.  Build it with
`python -m paper_1809_10786_b200.build`.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libsgl_b200.so")
# tests / tools only: SGL_LIBRARY=<path> loads another build of the same ABI
# (the bounds-checked libsgl_b200_checked.so, build.py --checked)
LIB_PATH = os.environ.get("SGL_LIBRARY", LIB_PATH)

SGL_OK, SGL_EINVAL, SGL_ECUDA, SGL_ENOMEM, SGL_EUNSUPPORTED = 0, 1, 2, 3, 4
FLAG_COMPACT_K1 = 1 << 0
FLAG_EXACT_LAST_STAGE = 1 << 1
FLAG_GENERIC_GRIDDING = 1 << 2
FLAG_PROFILE = 1 << 3
FLAG_PRECISE = 1 << 4
FLAG_FP64_WINDOW = 1 << 5
FLAG_I8_SCATTER = 1 << 6
FLAG_FP64_SCATTER = 1 << 7
FLAG_FULL_FFT = 1 << 8
FLAG_I8_GATHER = 1 << 9
FLAG_SCATTER_WIDE = 1 << 10
FLAG_SCATTER_NARROW = 1 << 11
FLAG_I8_PROF = 1 << 12
FLAG_NO_GUARD = 1 << 13
FLAG_FP64_TABLES = 1 << 14
FLAG_DETERMINISTIC = 1 << 15
STAGES = ("h2d", "basal", "fft", "window", "d2h")

# every symbol include/sgl_b200.h declares
EXPORTS = (
    "sgl_plan_create", "sgl_nfft_plan_create", "sgl_forward", "sgl_adjoint", "sgl_forward_adjoint", "sgl_direct_forward",
    "sgl_direct_adjoint", "sgl_plan_destroy", "sgl_plan_get_info",
    "sgl_plan_stage_ms", "sgl_last_error", "sgl_set_device", "sgl_device_count", "sgl_version",
    "sgl_plan_grid", "sgl_adjoint_spread", "sgl_adjoint_slab_fft", "sgl_adjoint_from_packed",
    "sgl_plan_create_multi", "sgl_plan_planes", "sgl_adjoint_axis0", "sgl_adjoint_from_eta",
)


class GridInfo(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("N0", ctypes.c_int32), ("N1", ctypes.c_int32), ("N2", ctypes.c_int32),
        ("N1p", ctypes.c_int32), ("N2p", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("plane_elems", ctypes.c_int64),
        ("crop1", ctypes.c_int32), ("crop2", ctypes.c_int32),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int32),
        ("M", ctypes.c_int64),
        ("rho", ctypes.c_double),
        ("sigma", ctypes.c_int32),
        ("q", ctypes.c_int32),
        ("n_axis", ctypes.c_int32 * 3),
        ("grid", ctypes.c_int32 * 3),
        ("sigma_axes", ctypes.c_int32 * 3),
        ("sigma_eff", ctypes.c_double * 3),
        ("lam", ctypes.c_double * 3),
        ("coeff_count", ctypes.c_int64),
        ("n_tiles", ctypes.c_int64),
        ("tile_nodes", ctypes.c_int64),
        ("tile_dmma", ctypes.c_int64),
        ("generic", ctypes.c_int32),
        ("exact", ctypes.c_int32),
        ("plan_ms", ctypes.c_double),
        ("i8_gather", ctypes.c_int32),
        ("i8_tiles", ctypes.c_int64),
        ("i8_ksteps", ctypes.c_int64),
        ("i8_scatter", ctypes.c_int32),
        ("i8_sksteps", ctypes.c_int64),
        ("guard", ctypes.c_int32),
        ("guard_ap", ctypes.c_double),
        ("guard_fwd_fallbacks", ctypes.c_int64),
        ("guard_adj_fallbacks", ctypes.c_int64),
        ("guard_est_fwd", ctypes.c_double),
        ("guard_est_adj", ctypes.c_double),
        ("n_gpus", ctypes.c_int32),
    ]


_LIB = None


class NativeLibraryError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load the CUDA library; raise loudly when it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1809_10786_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double
    L.sgl_plan_create.argtypes = [i32, i64, vp, i32, i32, dbl, u32, vp, ctypes.POINTER(vp)]
    L.sgl_plan_create.restype = ctypes.c_int
    L.sgl_plan_create_multi.argtypes = [i32, i64, vp, i32, i32, dbl, u32, i32, vp, ctypes.POINTER(vp)]
    L.sgl_plan_create_multi.restype = ctypes.c_int
    L.sgl_forward.argtypes = [vp, vp, i64, vp, vp]
    L.sgl_forward.restype = ctypes.c_int
    L.sgl_adjoint.argtypes = [vp, vp, vp, vp]
    L.sgl_adjoint.restype = ctypes.c_int
    L.sgl_nfft_plan_create.argtypes = [ctypes.c_int32, vp, ctypes.c_int64, vp, vp, ctypes.c_int32, ctypes.c_uint32,
                                       vp, vp]
    L.sgl_nfft_plan_create.restype = ctypes.c_int
    L.sgl_forward_adjoint.argtypes = [vp, vp, vp, vp, vp, vp]
    L.sgl_forward_adjoint.restype = ctypes.c_int
    for fn in (L.sgl_direct_forward, L.sgl_direct_adjoint):
        fn.argtypes = [ctypes.c_int32, ctypes.c_int64, vp, vp, vp, vp]
        fn.restype = ctypes.c_int
    L.sgl_plan_destroy.argtypes = [vp]
    L.sgl_plan_destroy.restype = None
    L.sgl_plan_get_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    L.sgl_plan_get_info.restype = ctypes.c_int
    L.sgl_plan_stage_ms.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_float), i32]
    L.sgl_plan_stage_ms.restype = ctypes.c_int
    L.sgl_last_error.argtypes = []
    L.sgl_last_error.restype = ctypes.c_char_p
    L.sgl_set_device.argtypes = [i32]
    L.sgl_set_device.restype = ctypes.c_int
    L.sgl_device_count.argtypes = [ctypes.POINTER(i32)]
    L.sgl_device_count.restype = ctypes.c_int
    L.sgl_plan_grid.argtypes = [vp, ctypes.POINTER(GridInfo)]
    L.sgl_plan_grid.restype = ctypes.c_int
    L.sgl_adjoint_spread.argtypes = [vp, vp, vp]
    L.sgl_adjoint_spread.restype = ctypes.c_int
    L.sgl_adjoint_slab_fft.argtypes = [vp, i32, i32, vp, vp]
    L.sgl_adjoint_slab_fft.restype = ctypes.c_int
    L.sgl_adjoint_from_packed.argtypes = [vp, vp, vp, vp]
    L.sgl_adjoint_from_packed.restype = ctypes.c_int
    L.sgl_plan_planes.argtypes = [vp, vp]
    L.sgl_plan_planes.restype = ctypes.c_int
    L.sgl_adjoint_axis0.argtypes = [vp, vp, i64, i64, vp, vp]
    L.sgl_adjoint_axis0.restype = ctypes.c_int
    L.sgl_adjoint_from_eta.argtypes = [vp, vp, vp, vp]
    L.sgl_adjoint_from_eta.restype = ctypes.c_int
    L.sgl_version.argtypes = []
    L.sgl_version.restype = ctypes.c_char_p
    _LIB = L
    return L


def check(rc: int) -> None:
    """Map C return codes to the reference's exception types."""
    if rc == SGL_OK:
        return
    msg = lib().sgl_last_error().decode() or f"error code {rc}"
    if rc in (SGL_EINVAL, SGL_EUNSUPPORTED):
        raise ValueError(msg)
    if rc == SGL_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    n = ctypes.c_int32(0)
    lib().sgl_device_count(ctypes.byref(n))
    return int(n.value)
