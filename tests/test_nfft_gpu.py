"""The NFFT layer on the device (sgl_nfft_plan_create + sgl_forward /
sgl_adjoint) against the reference's own nfft_execute / nfft_adjoint_execute
/ ndft / ndft_adjoint outputs (tests/golden/make_golden.py, nfft_cases)."""
import numpy as np
import pytest

from conftest import NFFT, load_golden

pytestmark = pytest.mark.gpu


def rel(x, ref):
    return float(np.max(np.abs(np.asarray(x) - ref)) / np.max(np.abs(ref)))


@pytest.fixture(scope="module")
def sgl():
    import paper_1809_10786_b200 as s
    return s


@pytest.mark.parametrize("backend", ["auto", "tiled", "generic"])
@pytest.mark.parametrize("name", NFFT)
def test_nfft_matches_reference(sgl, name, backend):
    g = load_golden(name)
    d = int(g["d"]) if "d" in g else 3
    n = tuple(int(v) for v in g["n"])
    sig = np.broadcast_to(g["sigma"], (d,))
    p = sgl.nfft_plan(d, n, tuple(int(s) for s in sig), int(g["q"]), g["nodes"], backend=backend)
    assert p.grid_shape == tuple(1 << int(np.ceil(np.log2(int(s) * k))) for s, k in zip(sig, n))
    assert rel(sgl.nfft_execute(p, g["coeffs"]), g["fwd"]) <= 1e-10
    assert rel(sgl.nfft_adjoint_execute(p, g["values"]), g["adj"]) <= 1e-10


@pytest.mark.parametrize("name", [n for n in NFFT if "ndft" in load_golden(n)])
def test_ndft_matches_reference(sgl, name):
    g = load_golden(name)
    d = int(g["d"]) if "d" in g else 3
    n = tuple(int(v) for v in g["n"])
    assert rel(sgl.ndft(d, n, g["coeffs"], g["nodes"]), g["ndft"]) <= 1e-12
    assert rel(sgl.ndft_adjoint(d, n, g["values"], g["nodes"]), g["ndft_adj"]) <= 1e-12


def test_nfft_pairing_torch_and_errors(sgl):
    import torch
    g = load_golden("nfft_d")
    n = tuple(int(v) for v in g["n"])
    p = sgl.nfft_plan(3, n, 2, 16, g["nodes"])
    f, v = g["coeffs"], g["values"]
    lhs = np.vdot(v, sgl.nfft_execute(p, f))
    rhs = np.vdot(sgl.nfft_adjoint_execute(p, v), f)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)   # the fast pair is an exact adjoint pair
    dev = torch.device("cuda", 0)
    fd = sgl.nfft_execute(p, torch.as_tensor(f, device=dev))
    assert fd.is_cuda and rel(fd.cpu().numpy(), g["fwd"]) <= 1e-10
    ad = sgl.nfft_adjoint_execute(p, torch.as_tensor(v, device=dev))
    assert ad.is_cuda and tuple(ad.shape) == n and rel(ad.cpu().numpy(), g["adj"]) <= 1e-10
    with pytest.raises(ValueError):
        sgl.nfft_execute(p, f[:, :, :-1])
    with pytest.raises(ValueError):
        sgl.nfft_adjoint_execute(p, v[:-1])


def test_sgl_basis_eval_matches_reference(sgl):
    g = load_golden("nfft_index")
    for t, ref in zip(g["basis_idx"], g["basis"]):
        assert rel(sgl.sgl_basis_eval(tuple(t), g["basis_pts"]), ref) <= 1e-12
    assert isinstance(sgl.sgl_basis_eval((2, 1, 0), [1.0, 0.5, 0.2]), complex)
