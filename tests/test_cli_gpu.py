"""The transform commands of the CLI on the device against files the
reference CLI wrote for the same inputs (tests/golden/csv/RUNS.txt)."""
import os

import numpy as np
import pytest

from paper_1809_10786_b200 import cli, csvio

pytestmark = pytest.mark.gpu

CSV = os.path.join(os.path.dirname(__file__), "golden", "csv")


def rel(x, ref):
    return float(np.max(np.abs(x - ref)) / np.max(np.abs(ref)))


@pytest.mark.parametrize("extra,name", [(["--method", "naive"], "f_naive.csv"), (["-q", "8"], "f_fast.csv"),
                                        (["--method", "fast-exact"], "f_exact.csv")])
def test_forward_command(tmp_path, extra, name):
    out = str(tmp_path / name)
    argv = ["forward", "--coeffs", os.path.join(CSV, "c_b5.csv"), "--points", os.path.join(CSV, "p_m40.csv"),
            "--out", out] + extra
    assert cli.main(argv) == 0
    assert rel(csvio.read_values(out), csvio.read_values(os.path.join(CSV, name))) <= 1e-12


@pytest.mark.parametrize("extra,name", [(["--method", "naive"], "a_naive.csv"), (["-q", "8"], "a_fast.csv")])
def test_adjoint_command(tmp_path, extra, name):
    out = str(tmp_path / name)
    argv = ["adjoint", "--values", os.path.join(CSV, "f_naive.csv"), "--points", os.path.join(CSV, "p_m40.csv"),
            "-B", "5", "--out", out] + extra
    assert cli.main(argv) == 0
    c, B = csvio.read_coeffs(out)
    ref, _ = csvio.read_coeffs(os.path.join(CSV, name))
    assert B == 5 and rel(c, ref) <= 1e-12


def test_invert_command(tmp_path, capsys):
    out = str(tmp_path / "inv.csv")
    argv = ["invert", "--values", os.path.join(CSV, "f_naive.csv"), "--points", os.path.join(CSV, "p_m40.csv"),
            "-B", "3", "--max-iter", "50", "--out", out]
    assert cli.main(argv) == 0
    assert "converged=True" in capsys.readouterr().out
    c, _ = csvio.read_coeffs(out)
    ref, _ = csvio.read_coeffs(os.path.join(CSV, "inv_b3.csv"))
    assert rel(c, ref) <= 1e-9


def _table(path):
    with open(path) as fh:
        lines = [ln.rstrip("\n") for ln in fh if ln.strip()]
    meta = lines[0]
    header = lines[1].split(",")
    rows = np.array([[float(x) for x in ln.split(",")] for ln in lines[2:]])
    return meta, header, rows


@pytest.mark.parametrize("name,argv", [
    ("exp_q.csv", ["experiment", "error-vs-q", "-B", "5", "-M", "80", "--kappa", "3.0", "--q-list", "2,4,8,12,16",
                   "--repetitions", "3", "--seed", "11"]),
    ("exp_radius.csv", ["experiment", "error-vs-radius", "-B", "4", "-M", "60", "--kappa-list", "0.5,2,4", "-q",
                        "10", "--repetitions", "2", "--seed", "12"]),
    ("exp_bw.csv", ["experiment", "error-vs-bandwidth", "--bandwidth-list", "3,6", "-M", "50", "--kappa", "2.5",
                    "-q", "8", "--repetitions", "2", "--seed", "13", "--exact-control"]),
    ("exp_inv.csv", ["experiment", "inverse-convergence", "-B", "3", "-q", "8", "--grid-n-list", "6", "--kappa",
                     "1.5", "--max-iter", "12", "--seed", "14"]),
])
def test_experiment_tables_match_reference(tmp_path, name, argv):
    """Same table layout (schema tags, columns, sweep keys) as the reference's
    run; error columns agree to the reference's own precision where the
    window error dominates rounding (> 1e-11), and stay at rounding level
    below that."""
    out = str(tmp_path / name)
    assert cli.main(argv + ["--out", out]) == 0
    m1, h1, r1 = _table(out)
    m0, h0, r0 = _table(os.path.join(CSV, name))
    assert m1 == m0 and h1 == h0 and r1.shape == r0.shape
    assert np.array_equal(r1[:, 0], r0[:, 0])
    if name == "exp_inv.csv":
        assert np.array_equal(r1[:, :3], r0[:, :3])
        np.testing.assert_allclose(r1[:8, 3:], r0[:8, 3:], rtol=1e-5)
        return
    for j, col in enumerate(h0):
        if not col.startswith("avg_max"):
            continue
        for a, b in zip(r1[:, j], r0[:, j]):
            if b > 1e-11:
                assert abs(a - b) <= 1e-2 * b, (col, a, b)
            else:
                assert a <= 1e-11, (col, a, b)


def test_runtime_experiment_table(tmp_path):
    out = str(tmp_path / "rt.csv")
    assert cli.main(["experiment", "runtime", "-B", "6", "--m-list", "10,200", "--repetitions", "2",
                     "--out", out]) == 0
    meta, header, rows = _table(out)
    assert header == ["M", "naive_mean_s", "naive_median_s", "fast_mean_s", "fast_median_s"]
    assert "kind=runtime" in meta and rows.shape == (2, 5) and np.all(rows[:, 1:] > 0)
