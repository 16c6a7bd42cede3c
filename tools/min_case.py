"""Minimal forward + adjoint on a small golden case (for compute-sanitizer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10786_b200 as sgl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "b8_q16"
backend = sys.argv[2] if len(sys.argv) > 2 else "auto"
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"ref_{name}.npz"))
p = sgl.plan(int(g["B"]), g["points"], q=int(g["q"]), rho=float(g["rho"]), compact_k1=bool(g["compact"]),
             backend=backend)
f = sgl.forward(p, g["coeffs"])
print("fwd", np.max(np.abs(f - g["fwd"])) / np.max(np.abs(g["fwd"])), flush=True)
a = sgl.adjoint(p, g["values"])
print("adj", np.max(np.abs(a - g["adj"])) / np.max(np.abs(g["adj"])), flush=True)
