"""B200-native NFSGLFT: forward / adjoint spherical Gauss-Laguerre transforms
at scattered points (arXiv 1809.10786), behind the reference `sglnufft`
surface `plan / forward / adjoint` (reference __init__.py:13-56).

The transform runs in `_lib/libsgl_b200.so` (sm_100a CUDA: FP64 DMMA window
kernels, bulk-async slab staging, cuFFT) via the C ABI `include/sgl_b200.h`.
There is no CPU fallback.
"""
from .generate import (cartesian_to_spherical, coeff_count, gen_coeffs, gen_grid,  # noqa: F401
                       gen_points_ball)
from .transform import (SglPlan, adjoint, choose_rho, evaluate_direct, evaluate_direct_adjoint,  # noqa: F401
                        forward, forward_adjoint, plan)

__all__ = [
    "SglPlan", "adjoint", "cartesian_to_spherical", "choose_rho", "coeff_count", "evaluate_direct",
    "evaluate_direct_adjoint", "forward", "forward_adjoint", "gen_coeffs", "gen_grid", "gen_points_ball", "plan",
]
__version__ = "0.1.0"
