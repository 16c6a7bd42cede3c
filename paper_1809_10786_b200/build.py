"""Build the in-tree CUDA library `libsgl_b200.so` for sm_100a.

    python -m paper_1809_10786_b200.build [--force]

Explicit nvcc (no JIT cache): the .so lands next to this file in `_lib/`
so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libsgl_b200.so")
SOURCES = ["capi.cu", "nodes.cu", "basal.cu", "gridding.cu", "gather_i8.cu", "scatter_i8.cu", "exact.cu", "direct.cu",
           "guard.cu", "dist.cu", "multi.cu", "determ.cu"]
HEADERS = ["sgl_internal.cuh", "umma.cuh", "i8_common.cuh", os.path.join("..", "..", "include", "sgl_b200.h")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


CHECKED_LIB = os.path.join(LIBDIR, "libsgl_b200_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False, variant: str | None = None,
          defines: tuple = ()) -> str:
    """checked=True: a separate library with device-side bounds checks
    (-DSGL_CHECKED, SGL_DCHECK in the kernels), loaded when SGL_LIBRARY points
    at it (tests/tools only); the product library never carries them.
    variant="name", defines=("-DX=1", ...): an experimental build in
    _lib/variants/ (kernel A/B measurements via SGL_LIBRARY)."""
    lib = CHECKED_LIB if checked else LIB
    if variant:
        lib = os.path.join(LIBDIR, "variants", f"libsgl_{variant}.so")
    if not force and not _stale(lib):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj_checked" if checked else "obj")
    if variant:
        objdir = os.path.join(LIBDIR, "variants", "obj_" + variant)
    os.makedirs(objdir, exist_ok=True)
    base = [nvcc()]
    # /usr/bin/g++ is the host compiler with a complete toolchain in this image
    if os.path.exists("/usr/bin/g++"):
        base += ["-ccbin", "/usr/bin/g++"]
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             "-I", os.path.join(HERE, "..", "include")] + (["-DSGL_CHECKED"] if checked else []) + list(defines)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        res = subprocess.run(base + flags + ["-c", os.path.join(CSRC, src), "-o", obj],
                             capture_output=True, text=True)
        return src, obj, res

    # one nvcc per translation unit, in parallel (the kernels are independent)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for src, obj, res in results:
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
        if verbose:
            sys.stderr.write(res.stderr)
    tmp = lib + ".tmp"
    res = subprocess.run(base + ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] +
                         [obj for _, obj, _ in results] + ["-lcufft", "-lpthread"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libsgl_b200.so")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_1809_10786_b200.build [--force] [-v] [--checked] [--variant NAME -DX=1 ...]
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv,
                variant=var, defines=tuple(a for a in sys.argv if a.startswith("-D"))))
