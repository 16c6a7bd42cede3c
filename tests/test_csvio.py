"""CSV formats and the command line (reference csvio.py, cli.py): files the
reference CLI wrote (tests/golden/csv/, tests/golden/make_golden.py) must be
reproduced byte for byte by the generators and round-trip through the
readers/writers here.  The transform commands run on the GPU
(tests/test_cli_gpu.py)."""
import os

import numpy as np
import pytest

from paper_1809_10786_b200 import cli, csvio

CSV = os.path.join(os.path.dirname(__file__), "golden", "csv")


def _bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("argv,name", [
    (["gen-coeffs", "-B", "5", "--seed", "7"], "c_b5.csv"),
    (["gen-points", "-M", "40", "--kappa", "2.5", "--seed", "3"], "p_m40.csv"),
    (["gen-grid", "-N", "4", "--kappa", "1.5"], "g_n4.csv"),
])
def test_generators_match_reference_files(tmp_path, argv, name):
    out = tmp_path / name
    assert cli.main(argv + ["--out", str(out)]) == 0
    assert _bytes(out) == _bytes(os.path.join(CSV, name))


@pytest.mark.parametrize("name,kind", [("c_b5.csv", "coeffs"), ("a_fast.csv", "coeffs"), ("inv_b3.csv", "coeffs"),
                                       ("p_m40.csv", "points"), ("g_n4.csv", "points"),
                                       ("f_naive.csv", "values"), ("f_exact.csv", "values")])
def test_read_write_round_trip_is_byte_exact(tmp_path, name, kind):
    src = os.path.join(CSV, name)
    out = str(tmp_path / name)
    if kind == "coeffs":
        c, B = csvio.read_coeffs(src)
        csvio.write_coeffs(out, c, B)
    elif kind == "points":
        csvio.write_points(out, csvio.read_points(src))
    else:
        csvio.write_values(out, csvio.read_values(src))
    assert _bytes(out) == _bytes(src)


def test_reader_errors_and_exit_codes(tmp_path, capsys):
    bad = tmp_path / "bad.csv"
    bad.write_text("# sglnufft-csv v1\nx,y,z\n1,2,3\n")
    with pytest.raises(ValueError):
        csvio.read_points(str(bad))
    with pytest.raises(ValueError):
        csvio.read_values(str(bad))
    with pytest.raises(ValueError):
        csvio.read_coeffs(str(bad))
    odd = tmp_path / "odd.csv"   # 4 rows: not a coefficient count
    odd.write_text("mu,n,l,m,re,im\n" + "".join(f"{i},1,0,0,0,0\n" for i in range(4)))
    with pytest.raises(ValueError):
        csvio.read_coeffs(str(odd))
    empty = tmp_path / "empty.csv"
    empty.write_text("# sglnufft-csv v1\n\n")
    with pytest.raises(ValueError):
        csvio.read_points(str(empty))
    # contract violations exit 1 with a message (reference cli.py:191-193)
    rc = cli.main(["forward", "--coeffs", str(tmp_path / "missing.csv"), "--points", str(bad),
                   "--out", str(tmp_path / "o.csv")])
    assert rc == 1 and "sglnufft: error:" in capsys.readouterr().err
    assert cli.main(["gen-points", "-M", "0", "--out", str(tmp_path / "o.csv")]) == 1
    assert not (tmp_path / "o.csv").exists()   # no partial output


def test_coefficient_rows_follow_mu_order():
    c, B = csvio.read_coeffs(os.path.join(CSV, "c_b5.csv"))
    assert B == 5 and c.shape == (55,)
    from paper_1809_10786_b200.generate import gen_coeffs, nlm_table
    np.testing.assert_array_equal(c, gen_coeffs(5, 7))
    t = nlm_table(3)
    assert t[0].tolist() == [1, 0, 0] and t[4].tolist() == [2, 1, 1] and t[5].tolist() == [3, 0, 0]


def test_experiment_spec_validation_and_paper_scale():
    from paper_1809_10786_b200.experiments import ExperimentSpec, paper_scale
    for kind in ("error-vs-q", "error-vs-radius", "error-vs-bandwidth", "runtime", "inverse-convergence"):
        with pytest.raises(ValueError):
            ExperimentSpec(kind=kind).validate()   # empty sweep list
    with pytest.raises(ValueError):
        ExperimentSpec(kind="nope").validate()
    with pytest.raises(ValueError):
        ExperimentSpec(kind="error-vs-q", q_list=[4], repetitions=0).validate()
    s = paper_scale(ExperimentSpec(kind="error-vs-bandwidth"))
    assert s.B_list == [8, 16, 32, 64, 128] and s.M == 1000 and s.q == 12
    s = paper_scale(ExperimentSpec(kind="inverse-convergence"))
    assert s.grid_n_list == [25, 50, 100] and s.max_iter == 10_000 and s.q == 15


def test_csv_table_render_matches_reference_layout():
    t = csvio.CsvTable(["q", "err"], [[4, 0.5], [8, 1e-20]], {"kind": "x", "B": 3})
    assert t.render() == "# sglnufft-csv v1 kind=x B=3\nq,err\n4,0.5\n8,9.9999999999999995e-21\n"
    with pytest.raises(ValueError):
        csvio.CsvTable(["a"], [[1, 2]]).render()
