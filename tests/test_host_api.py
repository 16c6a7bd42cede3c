"""Host-side mirror of the reference API: ValueError conditions raised before
any device work (transform.py:340-356, 385-402)."""
import numpy as np
import pytest

import paper_1809_10786_b200 as sgl


def pts(n=5, r=1.0):
    rng = np.random.default_rng(0)
    return sgl.gen_points_ball(n, r, rng)


@pytest.mark.parametrize("kw,msg", [
    (dict(B=0), "bandwidth"),
    (dict(B=2, q=16), "cutoff q = 16 must be below 4*sigma*B = 16"),
    (dict(B=4, q=0), "cutoff parameter q"),
    (dict(B=4, q=None), "cutoff parameter q"),
    (dict(B=4, rho=0.0), "rho must be positive"),
    (dict(B=4, rho=-1.0), "rho must be positive"),
    (dict(B=4, backend="fortran"), "backend"),
    (dict(B=4, q=20, backend="tiled"), "q <= 16"),
])
def test_plan_argument_errors(kw, msg):
    with pytest.raises(ValueError, match=msg.replace("*", r"\*")):
        sgl.plan(points=pts(), **kw)


def test_points_shape_rejected():
    with pytest.raises(ValueError, match="points must be"):
        sgl.plan(4, np.zeros((5, 2)))


def test_choose_rho_matches_reference():
    # test_transform.py:34-38
    p = np.array([[1.0, 0, 0], [5.0, 1, 2], [2.0, 2, 1]])
    assert sgl.choose_rho(p) == 5.0
    assert sgl.choose_rho(np.array([[0.0, 0, 0]])) == 1.0
