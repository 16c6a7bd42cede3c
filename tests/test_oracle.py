"""The CPU oracle is pinned against the reference: golden vectors produced by
running the reference package itself (tests/golden/make_golden.py) and the
reference's own known-answer values."""
import numpy as np
import pytest

from conftest import DIRECT, SMALL, load_golden
from oracle import sgl_oracle as o

TOL = 1e-12


@pytest.mark.parametrize("name", SMALL + ["cfg1", "cfg2_sub2000"])
def test_oracle_matches_reference_goldens(name, oracle_built):
    g = load_golden(name)
    p = o.oracle_plan(int(g["B"]), g["points"], q=int(g["q"]), rho=float(g["rho"]),
                      compact_k1=bool(g["compact"]))
    assert p.rho == float(g["rho"])
    f = o.oracle_forward(p, g["coeffs"])
    assert o.rel_linf(f, g["fwd"]) <= TOL
    a = o.oracle_adjoint(p, g["values"], threads=1)
    assert o.rel_linf(a, g["adj"]) <= TOL


@pytest.mark.parametrize("name", DIRECT)
def test_oracle_direct_sums_match_reference(name):
    # evaluate_direct(_adjoint) (transform.py:95-139) against the reference's own output
    g = load_golden(name)
    B = int(g["B"])
    assert o.rel_linf(o.evaluate_direct(g["coeffs"], B, g["points"]), g["fwd"]) <= TOL
    assert o.rel_linf(o.evaluate_direct_adjoint(g["values"], B, g["points"]), g["adj"]) <= TOL


def test_oracle_numpy_and_c_gridding_agree(oracle_built):
    # the TestBackends pattern (reference test_nfft.py:213-225)
    g = load_golden("b5_q10")
    p = o.oracle_plan(5, g["points"], q=10)
    rng = np.random.default_rng(0)
    grid = rng.normal(size=p.grid) + 1j * rng.normal(size=p.grid)
    a = o.gather(grid, p.base, p.win, p.q)
    saved, o._CLIB = o._CLIB, False
    try:
        b = o.gather(grid, p.base, p.win, p.q)
        sb = o.scatter(p.grid, p.base, p.win, g["values"], p.q)
    finally:
        o._CLIB = saved
    sa = o.scatter(p.grid, p.base, p.win, g["values"], p.q, threads=1)
    assert o.rel_linf(a, b) <= 1e-13
    assert o.rel_linf(sa, sb) <= 1e-13


def test_known_answers():
    # nfft.py geometry: lambda = 32 / (3 pi) for sigma = 2, q = 16 (test_nfft.py:75-80)
    grid, s_eff, lam = o.nfft_geometry((16,), (2,), 16)
    assert grid == (32,) and lam[0] == pytest.approx(32 / (3 * np.pi))
    d = o.deconv_factors((16, 16, 16), (32, 32, 32), (lam[0],) * 3)
    assert d[0][8] == pytest.approx(1.0)
    # grid (6, 10) -> (16, 32), sigma_eff = (16/6, 32/10) (test_nfft.py:82-86)
    grid, s_eff, _ = o.nfft_geometry((6, 10), (2, 2), 4)
    assert grid == (16, 32) and s_eff == pytest.approx((16 / 6, 32 / 10))
    # B = 1: f = c * pi^{-3/4} (test_transform.py:53-57)
    pts = np.array([[0.3, 1.0, 2.0], [1.1, 0.2, 5.0]])
    vals = o.evaluate_direct(np.array([2.0 - 1j]), 1, pts)
    assert vals == pytest.approx((2.0 - 1j) * np.pi ** -0.75)
    assert o.coeff_count(16) == 1496 and o.coeff_count(64) == 89440 and o.coeff_count(128) == 707264


@pytest.mark.parametrize("n", [3, 4, 8])
def test_fold_adjointness(n):
    rng = np.random.default_rng(n)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    y = rng.normal(size=2 * n) + 1j * rng.normal(size=2 * n)
    for f, ft in ((o.fold_even, o.fold_even_T), (o.fold_odd, o.fold_odd_T)):
        assert np.vdot(y, f(x)) == pytest.approx(np.vdot(ft(y), x), rel=1e-13, abs=1e-13)


def test_oracle_exact_stages_match_direct_sums():
    # basal factors are exact: with the exact last stage the staged pipeline
    # reproduces direct summation (test_transform.py:215-223)
    rng = np.random.default_rng(11)
    B = 4
    c = rng.uniform(-1, 1, o.coeff_count(B)) + 1j * rng.uniform(-1, 1, o.coeff_count(B))
    pts = np.column_stack([2.0 * rng.random(25) ** (1 / 3), np.arccos(rng.uniform(-1, 1, 25)),
                           rng.uniform(0, 2 * np.pi, 25)])
    p = o.oracle_plan(B, pts, q=8)
    eta = o.basal_forward(p, c)
    n = p.n_axis
    E = [np.exp(1j * np.outer(p.nodes[:, j], np.arange(n[j]) - n[j] // 2)) for j in range(3)]
    exact = np.einsum("abc,ma,mb,mc->m", eta, E[0], E[1], E[2])
    ref = o.evaluate_direct(c, B, pts)
    assert o.rel_linf(exact, ref) <= 1e-10


def test_extended_precision_truth_pinned():
    """oracle/extended.py (longdouble restatement of evaluate_direct_adjoint,
    transform.py:120-139) reproduces the reference's own direct sums, and the
    committed config-4 truth (tests/golden/make_truth.py) is consistent with
    the reference outputs it was measured against."""
    from oracle import extended as X
    for name in ("direct_b7", "direct_b16"):
        g = load_golden(name)
        t = X.direct_adjoint_ld(g["values"], int(g["B"]), g["points"], cos_fp64=True).astype(complex)
        assert o.rel_linf(t, g["adj"]) <= 1e-13
    t = load_golden("cfg4_truth")
    g = load_golden("cfg4_sub120")
    # the mpmath (60 digits) spot check of the longdouble truth
    assert float(np.max(t["mp_err"])) <= 1e-15
    # the reference fast adjoint's own error against the truth (2.56e-9: the
    # FP64 ill-conditioning of config 4, not a window error)
    assert o.rel_linf(g["adj"], t["truth"]) == pytest.approx(float(t["ref_fast_err"]), rel=1e-6)
    assert float(t["ref_direct_err"]) <= 1e-12
