"""Cost of the int8 accuracy guard per config-3 step: device time of forward +
adjoint with the guard on (default) and off (SGL_FLAG_NO_GUARD)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import _native, workloads
w = workloads.config(3)
dev = torch.device("cuda", 0)
pts, c, v = (torch.as_tensor(x, device=dev) for x in (w.points, w.coeffs, w.values))
for name, flags in (("guard on", 0), ("guard off", _native.FLAG_NO_GUARD)):
    p = sgl.plan(w.B, pts, flags=flags)
    for _ in range(3):
        sgl.forward(p, c); sgl.adjoint(p, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sgl.forward(p, c); sgl.adjoint(p, v)
    e1.record(); torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10:.3f} ms per forward + adjoint", flush=True)
    p.close()
