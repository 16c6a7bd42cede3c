import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1809_10786_b200 as sgl
g = np.load("/root/repo/tests/golden/ref_b12_q12.npz")
os.environ["SGL_GATHER"] = "i8"
p = sgl.plan(int(g["B"]), g["points"], q=int(g["q"]), rho=float(g["rho"]))
print("tiles", p.stats, flush=True)
f = sgl.forward(p, g["coeffs"])
print("dbg", os.environ.get("SGL_I8_DEBUG"), "rel", np.abs(f - g["fwd"]).max() / np.abs(g["fwd"]).max(), flush=True)
