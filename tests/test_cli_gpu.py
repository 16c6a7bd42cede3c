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
