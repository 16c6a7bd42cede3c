"""The device CG inverse against the reference's `invert` (solvers.py:204-277)
on the same inputs (goldens from the reference itself)."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solvers():
    from paper_1809_10786_b200 import _native, solvers as s
    assert _native.device_count() >= 1
    return s


def test_cgnr_matches_reference(solvers):
    g = load_golden("inv_cgnr_b4")
    rep = solvers.invert(g["points"], g["values"], int(g["B"]), max_iter=60, tol=1e-12, true_coeffs=g["coeffs"])
    assert rep.converged and bool(g["converged"])
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    sol = g["solution"]
    assert np.max(np.abs(rep.solution - sol)) <= 1e-9 * np.max(np.abs(sol))
    n = min(len(rep.residual_history), len(g["residual_history"]), 15)
    np.testing.assert_allclose(rep.residual_history[:n], g["residual_history"][:n], rtol=1e-6)
    assert rep.abs_error_history[-1] <= 1e-10


def test_cgne_matches_reference(solvers):
    g = load_golden("inv_cgne_b6")
    rep = solvers.invert(g["points"], g["values"], int(g["B"]), max_iter=40, tol=1e-12)
    assert rep.iterations == int(g["iterations"]) and rep.converged == bool(g["converged"])
    np.testing.assert_allclose(rep.residual_history[:20], g["residual_history"][:20], rtol=1e-6)


def test_midpoint_seed_and_cgnr_match_reference(solvers):
    # midpoint_initial_guess (solvers.py:166-191) by device direct sums, then CGNR from it
    g = load_golden("inv_mid_b4")
    B, kappa, N = int(g["B"]), float(g["kappa"]), int(g["grid_n"])
    x0 = solvers.midpoint_initial_guess(g["values"], g["points"], B, kappa, N)
    assert np.max(np.abs(x0 - g["x0"])) <= 1e-12 * np.max(np.abs(g["x0"]))
    rep = solvers.invert(g["points"], g["values"], B, x0_mode="midpoint", kappa=kappa, grid_n=N, max_iter=30,
                         tol=1e-12)
    assert rep.converged == bool(g["converged"]) and abs(rep.iterations - int(g["iterations"])) <= 1
    sol = g["solution"]
    assert np.max(np.abs(rep.solution - sol)) <= 1e-9 * np.max(np.abs(sol))
    with pytest.raises(ValueError):
        solvers.midpoint_initial_guess(g["values"], g["points"], B, kappa, N, weight="volume")


def test_operator_pairing_and_errors(solvers):
    import paper_1809_10786_b200 as sgl
    g = load_golden("b8_q16")
    op = solvers.operator_from_plan(sgl.plan(8, g["points"]))
    assert op.pairing_defect(g["coeffs"], g["values"]) <= 1e-12
    with pytest.raises(ValueError):
        solvers.invert(g["points"], g["values"], 8, solver="lsqr")
    with pytest.raises(ValueError):
        solvers.invert(g["points"], g["values"], 8, x0_mode="midpoint")
    with pytest.warns(UserWarning):
        solvers.invert(g["points"][:50], g["values"][:50], 8, solver="cgnr", max_iter=2)
