"""Print tile statistics of the gather / scatter plans for a BASELINE config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10786_b200 as sgl  # noqa: E402
from paper_1809_10786_b200 import workloads  # noqa: E402

for c, m in [(2, None), (3, None), (3, 2_000_000), (5, None)]:
    w = workloads.config(c, M=m)
    p = sgl.plan(w.B, w.points, rho=w.rho)
    st = p.stats
    print(c, w.M, "tiles", st["n_tiles"], "nodes/tile %.1f" % (w.M / st["n_tiles"]),
          "dmma/node %.0f" % (st["tile_dmma"] / w.M), "ideal 256", flush=True)
