"""e2e of sgl_forward_adjoint at config 3 with pinned vs pageable host buffers,
and the batched forward into host memory (config 5 shape) pinned vs pageable,
against the device-only time of the same calls."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import workloads

def timeit(fn, n=5):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3

w = workloads.config(3)
p = sgl.plan(w.B, w.points)
dev = torch.device("cuda", 0)
cd, vd = torch.as_tensor(w.coeffs, device=dev), torch.as_tensor(w.values, device=dev)
print("cfg3 device  %.2f ms" % timeit(lambda: sgl.forward_adjoint(p, cd, vd)), flush=True)
pin = lambda a: (lambda t: (t.numpy().__setitem__(slice(None), a), t.numpy())[1])(torch.empty(a.shape, dtype=torch.complex128, pin_memory=True))
cp, vp = pin(w.coeffs), pin(w.values)
print("cfg3 pinned   %.2f ms" % timeit(lambda: sgl.forward_adjoint(p, cp, vp)), flush=True)
print("cfg3 pageable %.2f ms" % timeit(lambda: sgl.forward_adjoint(p, w.coeffs, w.values)), flush=True)
p.close()
w5 = workloads.config(5, M=500_000)
p5 = sgl.plan(w5.B, w5.points)
C = w5.coeffs[:16]
Cd = torch.as_tensor(C, device=dev)
print("cfg5x16 device   %.2f ms" % timeit(lambda: sgl.forward(p5, Cd), 3), flush=True)
print("cfg5x16 pageable %.2f ms" % timeit(lambda: sgl.forward(p5, C), 3), flush=True)
