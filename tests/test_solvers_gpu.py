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


@pytest.mark.parametrize("name,solver,it", [("inv_cgnr_b4", "cgnr", 60), ("inv_cgne_b6", "cgne", 40)])
def test_graph_iterations_match_eager(solvers, name, solver, it):
    """The CUDA-graph CG (scalars on the device, batched replays, gated
    iterations past the stop) gives the eager loop's iteration count,
    solution, residual and error histories."""
    g = load_golden(name)
    B = int(g["B"])
    kw = dict(max_iter=it, tol=1e-12, solver=solver, true_coeffs=g.get("coeffs"))
    eager = solvers.invert(g["points"], g["values"], B, graph=False, **kw)
    graph = solvers.invert(g["points"], g["values"], B, graph=True, **kw)
    # The adjoint's atomic summation order makes any two runs differ in the last
    # bits, which CG amplifies near convergence (as against the reference's own
    # CPU run): compare like test_cgnr_matches_reference does.
    assert abs(graph.iterations - eager.iterations) <= 1 and graph.converged == eager.converged
    sol = eager.solution
    if eager.converged:   # (the CGNE case stops at max_iter, where the runs have drifted apart)
        assert np.max(np.abs(graph.solution - sol)) <= 1e-9 * np.max(np.abs(sol))
    assert len(graph.residual_history) == graph.iterations + 1
    n = min(len(graph.residual_history), len(eager.residual_history), 15)
    np.testing.assert_allclose(graph.residual_history[:n], eager.residual_history[:n], rtol=1e-6)
    assert len(graph.abs_error_history) == len(graph.rel_error_history) == graph.iterations + 1
    np.testing.assert_allclose(graph.abs_error_history[:n], eager.abs_error_history[:n], rtol=1e-6)
    np.testing.assert_allclose(graph.rel_error_history[:n], eager.rel_error_history[:n], rtol=1e-6)
    if eager.converged:
        assert graph.abs_error_history[-1] <= 1e-9 * np.max(np.abs(g["coeffs"]))


def test_graph_iteration_cap_and_operator_api(solvers):
    """tol = 0 runs exactly max_iter iterations (not a multiple of the replay
    batch); cgnr / cgne on an operator choose the graph path themselves; a
    plan with the int8 scatter (host-side accuracy guard) keeps the eager loop."""
    import paper_1809_10786_b200 as sgl
    g = load_golden("inv_cgnr_b4")
    B = int(g["B"])
    for m in (1, 7, solvers.GRAPH_BATCH + 3):
        a = solvers.invert(g["points"], g["values"], B, max_iter=m, tol=0.0, graph=False)
        b = solvers.invert(g["points"], g["values"], B, max_iter=m, tol=0.0, graph=True)
        assert a.iterations == b.iterations == m and not b.converged
        assert len(b.residual_history) == m + 1
        if m <= 7:   # before the runs' last-bit differences grow
            assert np.max(np.abs(a.solution - b.solution)) <= 1e-10 * np.max(np.abs(a.solution))
    op = solvers.operator_from_plan(sgl.plan(B, g["points"]))
    assert solvers._graph_eligible(op, False, None)
    assert not solvers._graph_eligible(op, True, None) and not solvers._graph_eligible(op, False, print)
    r1 = solvers.cgnr(op, g["values"], max_iter=solvers.GRAPH_MIN_ITERS, tol=1e-12)   # automatic: graph
    r2 = solvers.cgnr(op, g["values"], max_iter=solvers.GRAPH_MIN_ITERS, tol=1e-12, graph=False)
    assert abs(r1.iterations - r2.iterations) <= 1 and r1.converged and r2.converged
    r3 = solvers.cgne(op, g["values"], max_iter=5, graph=True)
    r4 = solvers.cgne(op, g["values"], max_iter=5)
    assert r3.iterations == r4.iterations and np.allclose(r3.residual_history, r4.residual_history, rtol=1e-8)
    rng = np.random.default_rng(5)
    p8 = sgl.plan(8, sgl.gen_points_ball(3000, 3.0, rng), backend="i8")
    assert p8.stats["i8_scatter"] and not solvers._graph_eligible(solvers.operator_from_plan(p8), False, None)
