"""Host-side pieces of the NFFT layer and the public helpers: the closed-form
bounds, basis indexing, the point warp, and the argument checks that run
before any device work (reference test_nfft.py / test_indexing.py idioms)."""
import numpy as np
import pytest

import paper_1809_10786_b200 as sgl
from conftest import load_golden


def test_nfft_error_bound_known_answer():
    # reference test_nfft.py:251-261
    assert sgl.nfft_error_bound(3, 2, 16, 1) == pytest.approx(7.072896720691885e-10, rel=1e-14)
    assert sgl.nfft_error_bound(3, 2, 16, 2.0) == pytest.approx(2 * 7.072896720691885e-10, rel=1e-14)
    with pytest.raises(ValueError):
        sgl.nfft_error_bound(3, 1, 16, 1)
    assert sgl.nfft_error_bound(3, 2, 12, 1) > sgl.nfft_error_bound(3, 2, 16, 1)


def test_error_bound_trends():
    assert sgl.error_bound(16, 3.0, 12, 1.0) > sgl.error_bound(16, 3.0, 16, 1.0)
    assert sgl.error_bound(32, 3.0, 16, 1.0) > sgl.error_bound(16, 3.0, 16, 1.0)
    with pytest.raises(ValueError):
        from paper_1809_10786_b200.transform import growth_threshold
        growth_threshold(1.5)


def test_indexing_matches_reference_table():
    g = load_golden("nfft_index")
    nlm = g["nlm"]
    assert np.array_equal(sgl.indexing.mu_to_nlm_array(10), nlm)
    for mu in range(len(nlm)):
        assert tuple(sgl.mu_to_nlm(mu, 10)) == tuple(nlm[mu])
        assert sgl.nlm_to_mu(*nlm[mu]) == mu
    with pytest.raises(ValueError):
        sgl.nlm_to_mu(2, 2, 0)
    with pytest.raises(ValueError):
        sgl.mu_to_nlm(sgl.coeff_count(10), 10)


def test_transform_points():
    pts = np.array([[0.0, 1.0, 2.0], [2.0, 0.5, 0.1], [1.0, np.pi, 0.0]])
    t = sgl.transform_points(pts, 2.0)
    assert t[0, 0] == pytest.approx(np.pi) and t[1, 0] == 0.0 and t[2, 0] == pytest.approx(np.pi / 2)
    assert np.array_equal(t[:, 1:], pts[:, 1:])
    with pytest.raises(ValueError):
        sgl.transform_points(pts, 1.0)


@pytest.mark.parametrize("kw,msg", [
    (dict(d=4), "d <= 3"), (dict(n_axis=(8, 9, 6)), "even"), (dict(sigma=1), "oversampling"),
    (dict(q=0), "cutoff"), (dict(q=32, n_axis=(8, 8, 8)), "below sigma"), (dict(sigma=(2, 1, 2)), "oversampling"),
])
def test_nfft_plan_argument_errors(kw, msg):
    args = dict(d=3, n_axis=(8, 10, 6), sigma=2, q=6, nodes=np.zeros((4, 3)))
    args.update(kw)
    if args["d"] != 3:
        args["nodes"] = np.zeros((4, args["d"]))
    with pytest.raises(ValueError, match=msg):
        sgl.nfft_plan(args["d"], args["n_axis"], args["sigma"], args["q"], args["nodes"])
