"""The input generators restate the reference's draw order exactly (pinned
against inputs the reference generated, tests/golden/make_golden.py)."""
import numpy as np

from conftest import load_golden
from paper_1809_10786_b200 import workloads
from paper_1809_10786_b200.generate import coeff_count, gen_coeffs, gen_grid


def test_config1_inputs_match_reference():
    g = load_golden("cfg1")
    w = workloads.config(1)
    assert np.array_equal(w.points, g["points"])
    assert np.array_equal(w.coeffs, g["coeffs"])
    assert np.array_equal(w.values, g["values"])
    assert w.rho == float(g["rho"])


def test_config2_subset_matches_reference():
    g = load_golden("cfg2_sub2000")
    w = workloads.config(2)
    sel, ws = workloads.subset(w, 2000)
    assert np.array_equal(sel, g["sel"])
    assert np.array_equal(ws.points, g["points"])
    assert np.array_equal(ws.values, g["values"])
    assert np.array_equal(w.coeffs, g["coeffs"])
    assert ws.rho == float(g["rho"])


def test_config3_and_5_heads_match_reference():
    g3 = load_golden("cfg3_sub600")
    w3 = workloads.config(3)
    assert np.array_equal(w3.coeffs, g3["coeffs"])
    assert np.array_equal(w3.points[:8], g3["head"])
    assert np.array_equal(w3.values[:8], g3["vhead"])
    sel, ws = workloads.subset(w3, 600)
    assert np.array_equal(sel, g3["sel"]) and np.array_equal(ws.points, g3["points"])
    assert ws.rho == float(g3["rho"])
    del w3, ws
    g5 = load_golden("cfg5_sub400")
    w5 = workloads.config(5, M=2_000_000)
    assert np.array_equal(w5.points[:8], g5["head"])
    assert np.array_equal(w5.coeffs[[0, 63]], g5["coeffs"])
    assert np.array_equal(w5.points[g5["sel"]], g5["points"])


def test_counts_and_grid():
    assert coeff_count(16) == 1496
    assert gen_coeffs(3, 0).shape == (14,)
    pts = gen_grid(4, 1.0)
    assert pts.shape == (64, 3) and np.all(pts[:, 2] >= 0) and np.all(pts[:, 2] < 2 * np.pi)


def test_round2_subsets_match_reference():
    """The SURVEY 8(d)-sized subsets (tests/golden/make_golden.py scale_cases):
    config 3 and config 5 coefficients are not stored, only fingerprints of
    the reference's draw; the package's generators must reproduce them."""
    g3 = load_golden("cfg3_sub20k")
    w3 = workloads.config(3)
    assert np.array_equal(w3.coeffs[:64], g3["c_head"])
    assert np.allclose([w3.coeffs.sum(), np.abs(w3.coeffs).sum()], g3["c_sum"], rtol=1e-14, atol=0)
    sel, ws = workloads.subset(w3, 20_000, seed=2)
    assert np.array_equal(sel, g3["sel"]) and np.array_equal(ws.points, g3["points"])
    assert np.array_equal(ws.values, g3["values"]) and ws.rho == float(g3["rho"])
    del w3, ws
    g2 = load_golden("cfg2_sub20k")
    w2 = workloads.config(2)
    sel, ws = workloads.subset(w2, 20_000, seed=2)
    assert np.array_equal(sel, g2["sel"]) and np.array_equal(ws.points, g2["points"])
    assert np.array_equal(w2.coeffs, g2["coeffs"]) and np.array_equal(ws.values, g2["values"])
    w5 = workloads.config(5)
    for name, seed, k in (("cfg5_sub2k_all64", 2, 2_000), ("cfg5_sub20k_4v", 3, 20_000)):
        g5 = load_golden(name)
        assert np.array_equal(w5.coeffs[:, :16], g5["c_head"])
        assert np.allclose(np.stack([w5.coeffs.sum(axis=1), np.abs(w5.coeffs).sum(axis=1)], axis=1), g5["c_sum"],
                           rtol=1e-14, atol=0)
        sel, ws = workloads.subset(w5, k, seed=seed)
        assert np.array_equal(sel, g5["sel"]) and np.array_equal(ws.points, g5["points"])
        assert ws.rho == float(g5["rho"])
