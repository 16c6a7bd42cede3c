import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1809_10786_b200 as sgl
sys.path.insert(0, "/root/repo/tests")
from conftest import load_golden
for name in ["nfft_d", "nfft_b", "nfft_a", "nfft_c", "nfft_e"]:
    g = load_golden(name)
    d = int(g["d"]) if "d" in g else 3
    n = tuple(int(v) for v in g["n"]); sig = tuple(int(s) for s in np.broadcast_to(g["sigma"], (d,)))
    pa = sgl.nfft_plan(d, n, sig, int(g["q"]), g["nodes"])
    pt = sgl.nfft_plan(d, n, sig, int(g["q"]), g["nodes"], backend="tiled")
    fa, ft = sgl.nfft_execute(pa, g["coeffs"]), sgl.nfft_execute(pt, g["coeffs"])
    e = np.abs(fa - ft) / np.abs(ft).max()
    i = np.argsort(e)[::-1][:3]
    print(name, pa.backend, "n", n, "grid", pa.grid_shape, "q", int(g["q"]), "max rel", e.max(), "worst nodes", g["nodes"][i], e[i])
