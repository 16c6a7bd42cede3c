"""The C ABI from C alone (tests/c_abi/sgl_c_smoke.c): compiled and linked
against include/sgl_b200.h and the in-tree libsgl_b200.so on CPU; run on the
GPU (pairing, fast vs the device direct sums, the ValueError path, a
multi-device plan)."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "c_abi", "sgl_c_smoke.c")
LIBDIR = os.path.join(ROOT, "paper_1809_10786_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "sgl_c_smoke")
    r = subprocess.run(["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", SRC, "-I", os.path.join(ROOT, "include"),
                        "-L", LIBDIR, "-lsgl_b200", "-lm", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_compiles_and_links_against_the_abi(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_program_runs(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "C ABI smoke: OK" in r.stdout
