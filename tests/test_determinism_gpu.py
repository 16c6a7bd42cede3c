"""Deterministic adjoint (plan(..., deterministic=True), SGL_FLAG_DETERMINISTIC,
csrc/determ.cu).

The reference's spreading loop is serial (_gridding.py:77-95), so its adjoint
is bitwise reproducible; the default window kernels here reduce with FP64
atomics and agree run to run only to ~1e-13.  Under the flag every window
kernel (int8 scatter, FP64 DMMA scatter, per-node scatter) reduces 64-bit
fixed-point integers, so repeated adjoints must be bit-identical -- and still
within the parity bar of the reference's own outputs.
"""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
TOL = 1e-10        # parity bar against the reference goldens (test_parity_gpu.py)
TOL_SAME = 1e-12   # deterministic vs default plan of the same engine (fixed-point rounding: ~2^-60)


def rel(x, ref):
    x, ref = np.asarray(x), np.asarray(ref)
    return float(np.max(np.abs(x - ref)) / np.max(np.abs(ref)))


@pytest.fixture(scope="module")
def sgl():
    import paper_1809_10786_b200 as m
    return m


def _plan(sgl, g, **kw):
    return sgl.plan(int(g["B"]), g["points"], q=int(g["q"]), rho=float(g["rho"]),
                    compact_k1=bool(g["compact"]), **kw)


def _bitwise_repeat(sgl, p, v, n=4):
    outs = [sgl.adjoint(p, v) for _ in range(n)]
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint64), outs[0].view(np.uint64))
    return outs[0]


@pytest.mark.parametrize("backend", ["auto", "tiled", "generic", "i8"])
@pytest.mark.parametrize("name", ["b8_q16", "b12_q12", "b6_q6_compact", "edges_b4_q5", "cfg2_sub20k",
                                  "cfg3_sub20k"])
def test_deterministic_adjoint_bitwise_and_parity(sgl, name, backend):
    g = load_golden(name)
    if backend == "generic" and name.startswith("cfg"):
        pytest.skip("per-node kernels cross-checked on the small shapes")
    p = _plan(sgl, g, backend=backend, deterministic=True)
    a = _bitwise_repeat(sgl, p, g["values"])
    assert rel(a, g["adj"]) <= TOL, rel(a, g["adj"])
    a0 = sgl.adjoint(_plan(sgl, g, backend=backend), g["values"])
    assert rel(a, a0) <= TOL_SAME, rel(a, a0)


def test_deterministic_int8_scatter_at_scale(sgl):
    # 3e5 nodes on the int8 tensor-core scatter (512-node tiles, many CTAs per cell)
    rng = np.random.default_rng(11)
    pts = sgl.gen_points_ball(300_000, 6.0, rng)
    v = rng.standard_normal(len(pts)) + 1j * rng.standard_normal(len(pts))
    p = sgl.plan(32, pts, rho=6.5, backend="i8", deterministic=True)
    assert p.stats["i8_scatter"]
    a = _bitwise_repeat(sgl, p, v, n=3)
    a64 = sgl.adjoint(sgl.plan(32, pts, rho=6.5, backend="tiled"), v)
    assert rel(a, a64) <= 1e-11, rel(a, a64)
    # the FP64 DMMA scatter (the guard's fallback engine) under the flag
    pf = sgl.plan(32, pts, rho=6.5, backend="tiled", deterministic=True)
    af = _bitwise_repeat(sgl, pf, v, n=3)
    assert rel(af, a64) <= TOL_SAME, rel(af, a64)


@pytest.mark.parametrize("backend", ["auto", "tiled", "i8"])
@pytest.mark.parametrize("scale", [1e-300, 1e-30, 1e30, 1e300])
def test_deterministic_dynamic_range(sgl, backend, scale):
    # the fixed-point exponent spans the FP64 range (2^E applied as two exact factors)
    rng = np.random.default_rng(5)
    pts = sgl.gen_points_ball(4000, 4.0, rng)
    v = (rng.standard_normal(4000) + 1j * rng.standard_normal(4000)) * scale
    p = sgl.plan(16, pts, backend=backend, deterministic=True)
    a = _bitwise_repeat(sgl, p, v, n=2)
    assert np.all(np.isfinite(a))
    a64 = sgl.adjoint(sgl.plan(16, pts, backend="tiled"), v)
    assert rel(a, a64) <= 1e-11, rel(a, a64)


@pytest.mark.parametrize("backend", ["auto", "tiled", "i8"])
def test_deterministic_zero_and_nonfinite(sgl, backend):
    rng = np.random.default_rng(6)
    pts = sgl.gen_points_ball(3000, 4.0, rng)
    p = sgl.plan(12, pts, backend=backend, deterministic=True)
    assert np.all(sgl.adjoint(p, np.zeros(3000, complex)) == 0)
    v = rng.standard_normal(3000) + 0j
    v[17] = np.nan   # NaN + 0i
    assert np.isnan(sgl.adjoint(p, v)).any()   # NaN propagates (FP64 REDs for non-finite input)
    v[17] = 1j * np.inf
    assert not np.all(np.isfinite(sgl.adjoint(p, v)))
    v[17] = 1.0   # and the plan recovers on the next finite call
    a = _bitwise_repeat(sgl, p, v, n=2)
    assert np.all(np.isfinite(a))


def test_deterministic_forward_unchanged(sgl):
    # the flag touches only the adjoint's reduction; the forward has no atomics
    g = load_golden("b12_q12")
    f1 = sgl.forward(_plan(sgl, g, deterministic=True), g["coeffs"])
    f0 = sgl.forward(_plan(sgl, g), g["coeffs"])
    assert np.array_equal(f1, f0)
