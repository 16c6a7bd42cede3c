"""B200-native NFSGLFT: forward / adjoint spherical Gauss-Laguerre transforms
at scattered points (arXiv 1809.10786), behind the reference `sglnufft`
surface `plan / forward / adjoint` (reference __init__.py:13-56).

The transform runs in `_lib/libsgl_b200.so` (sm_100a CUDA: FP64 DMMA window
kernels, bulk-async slab staging, cuFFT) via the C ABI `include/sgl_b200.h`.
There is no CPU fallback.
"""
from .generate import (cartesian_to_spherical, coeff_count, gen_coeffs, gen_grid,  # noqa: F401
                       gen_points_ball)
from .indexing import SglIndex, mu_to_nlm, nlm_to_mu  # noqa: F401
from .nfft import (NfftPlan, ndft, ndft_adjoint, nfft_adjoint_execute, nfft_error_bound,  # noqa: F401
                   nfft_execute, nfft_plan)
from .solvers import (LinearOperatorPair, SolveReport, cgne, cgnr, invert,  # noqa: F401
                      midpoint_initial_guess, operator_from_plan)
from .transform import (SglPlan, adjoint, choose_rho, error_bound, evaluate_direct,  # noqa: F401
                        evaluate_direct_adjoint, forward, forward_adjoint, plan, sgl_basis_eval, transform_points)

__all__ = [
    "LinearOperatorPair", "NfftPlan", "SglIndex", "SglPlan", "SolveReport", "adjoint", "cartesian_to_spherical",
    "cgne", "cgnr", "choose_rho", "coeff_count", "error_bound", "evaluate_direct", "evaluate_direct_adjoint", "forward",
    "forward_adjoint", "gen_coeffs", "gen_grid", "gen_points_ball", "invert", "midpoint_initial_guess",
    "mu_to_nlm", "ndft", "ndft_adjoint", "nfft_adjoint_execute", "nfft_error_bound", "nfft_execute", "nfft_plan",
    "nlm_to_mu", "operator_from_plan", "plan", "sgl_basis_eval", "transform_points",
]
__version__ = "0.1.0"
