"""The C-ABI library loads on CPU and exports every symbol include/sgl_b200.h
declares; argument validation that happens before any device work returns the
reference's ValueError conditions."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1809_10786_b200 import _native


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sgl_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*\*?\s*(sgl_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 10
    lib = _native.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_version_and_device_count():
    assert b"sm_100a" in _native.lib().sgl_version()
    assert _native.device_count() >= 0


@pytest.mark.parametrize("B,M,sigma,q,flags,msg", [
    (0, 1, 2, 16, 0, "bandwidth must be >= 1"),
    (4, 1, 2, 0, 0, "cutoff parameter q must be >= 1"),
    (2, 1, 2, 16, 0, "cutoff q = 16 must be below 4*sigma*B = 16"),
    (4, 1, 1, 4, 0, "oversampling factor must be an integer >= 2"),
])
def test_plan_create_rejects_like_reference(B, M, sigma, q, flags, msg):
    lib = _native.lib()
    pts = (ctypes.c_double * 3)(1.0, 0.5, 0.5)
    h = ctypes.c_void_p(0)
    rc = lib.sgl_plan_create(B, M, ctypes.cast(pts, ctypes.c_void_p), sigma, q, 0.0, flags, None, ctypes.byref(h))
    assert rc in (_native.SGL_EINVAL, _native.SGL_EUNSUPPORTED)
    assert msg in lib.sgl_last_error().decode()
    assert not h.value
    with pytest.raises(ValueError):
        _native.check(rc)


def test_plan_info_layout_matches_header(tmp_path):
    # the ctypes mirror of sgl_plan_info must match the C struct field by field
    # (size and offsets from the header, compiled with the host C compiler)
    fields = [f[0] for f in _native.PlanInfo._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "sgl_b200.h"\nint main(void){\n'
                   '  printf("%zu\\n", sizeof(sgl_plan_info));\n' +
                   "".join(f'  printf("%zu\\n", offsetof(sgl_plan_info, {f}));\n' for f in fields) + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    rc = os.system(f"gcc -I{os.path.join(ROOT, 'include')} -o {exe} {src} 2>/dev/null")
    if rc != 0:
        pytest.skip("no host C compiler")
    got = [int(x) for x in os.popen(str(exe)).read().split()]
    assert got[0] == ctypes.sizeof(_native.PlanInfo)
    assert got[1:] == [getattr(_native.PlanInfo, f).offset for f in fields]
