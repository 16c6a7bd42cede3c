"""Direct summation on the device (sgl_direct_forward / sgl_direct_adjoint)
against the reference's evaluate_direct(_adjoint) (transform.py:95-139):
golden vectors produced by the reference, the oracle restatement at larger
B, and the fast transform."""
import numpy as np
import pytest

from conftest import DIRECT, load_golden

pytestmark = pytest.mark.gpu

TOL = 1e-12   # measured <= 5e-14 against the reference and the oracle (B <= 64)


def rel(x, ref):
    return float(np.max(np.abs(np.asarray(x) - ref)) / np.max(np.abs(ref)))


@pytest.fixture(scope="module")
def sgl():
    import paper_1809_10786_b200 as s
    return s


@pytest.mark.parametrize("name", DIRECT)
def test_direct_matches_reference(sgl, name):
    g = load_golden(name)
    B = int(g["B"])
    assert rel(sgl.evaluate_direct(g["coeffs"], B, g["points"]), g["fwd"]) <= TOL
    assert rel(sgl.evaluate_direct_adjoint(g["values"], B, g["points"]), g["adj"]) <= TOL


@pytest.mark.parametrize("B,M", [(40, 200), (64, 40)])
def test_direct_matches_oracle(sgl, B, M):
    from oracle import sgl_oracle as o
    rng = np.random.default_rng(B)
    c = sgl.gen_coeffs(B, rng)
    pts = sgl.gen_points_ball(M, 6.0, rng)
    v = rng.uniform(-1, 1, M) + 1j * rng.uniform(-1, 1, M)
    assert rel(sgl.evaluate_direct(c, B, pts), o.evaluate_direct(c, B, pts)) <= TOL
    assert rel(sgl.evaluate_direct_adjoint(v, B, pts), o.evaluate_direct_adjoint(v, B, pts)) <= TOL


def test_direct_pairing_and_fast_transform(sgl):
    # <F c, v> = <c, F^H v> for the direct pair; the fast pair (q = 16)
    # approximates it (reference test_transform.py:215-223 idiom)
    g = load_golden("cfg3_sub600")
    B = int(g["B"])
    pts, c, v = g["points"][:200], g["coeffs"], g["values"][:200]
    f = sgl.evaluate_direct(c, B, pts)
    a = sgl.evaluate_direct_adjoint(v, B, pts)
    lhs, rhs = np.vdot(v, f), np.vdot(a, c)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(f) * np.linalg.norm(v)
    p = sgl.plan(B, pts, rho=float(g["rho"]))
    assert rel(sgl.forward(p, c), f) <= 1e-8
    assert rel(sgl.adjoint(p, v), a) <= 1e-8


def test_direct_torch_errors_and_empty(sgl):
    import torch
    g = load_golden("direct_b7")
    dev = torch.device("cuda", 0)
    f = sgl.evaluate_direct(torch.as_tensor(g["coeffs"], device=dev), 7, torch.as_tensor(g["points"], device=dev))
    assert f.is_cuda and rel(f.cpu().numpy(), g["fwd"]) <= TOL
    a = sgl.evaluate_direct_adjoint(torch.as_tensor(g["values"], device=dev), 7, g["points"])
    assert a.is_cuda and rel(a.cpu().numpy(), g["adj"]) <= TOL
    with pytest.raises(ValueError):
        sgl.evaluate_direct(g["coeffs"][:-1], 7, g["points"])
    with pytest.raises(ValueError):
        sgl.evaluate_direct_adjoint(g["values"][:-1], 7, g["points"])
    with pytest.raises(ValueError):
        sgl.evaluate_direct(g["coeffs"], 0, g["points"])
    assert sgl.evaluate_direct(g["coeffs"], 7, np.zeros((0, 3))).shape == (0,)
    assert np.all(sgl.evaluate_direct_adjoint(np.zeros(0), 7, np.zeros((0, 3))) == 0)
