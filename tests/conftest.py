"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree CUDA library;
`-m "not gpu"` tests run on CPU (oracle pins, host logic, ABI exports)."""
import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsgl_b200.so")


def load_golden(name):
    d = np.load(os.path.join(GOLDEN, f"ref_{name}.npz"), allow_pickle=False)
    return {k: d[k] for k in d.files}


def golden_names(pattern="*"):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, f"ref_{pattern}.npz"))):
        out.append(os.path.basename(p)[4:-4])
    return out


SMALL = [n for n in golden_names() if not n.startswith(("cfg", "inv_", "direct_", "nfft_", "precise_"))]
NFFT = [n for n in golden_names() if n.startswith("nfft_") and n != "nfft_index"]
DIRECT = [n for n in golden_names() if n.startswith("direct_")]


@pytest.fixture(scope="session")
def oracle_built():
    """Build the C restatement of the window loops (test infrastructure)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    return True


@pytest.fixture(scope="session", autouse=True)
def native_built():
    """(Re)build libsgl_b200.so if any source is newer (no-op otherwise)."""
    from paper_1809_10786_b200 import build
    return build.build()
