"""Do two plans' forward and adjoint overlap usefully on two streams?"""
import torch

import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import workloads

w = workloads.config(3)
pts = torch.as_tensor(w.points, device="cuda")
c = torch.as_tensor(w.coeffs, device="cuda")
v = torch.as_tensor(w.values, device="cuda")
p1 = sgl.plan(w.B, pts, rho=w.rho)
p2 = sgl.plan(w.B, pts, rho=w.rho)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def seq():
    sgl.forward(p1, c)
    sgl.adjoint(p1, v)


def conc():
    with torch.cuda.stream(s1):
        sgl.forward(p1, c)
    with torch.cuda.stream(s2):
        sgl.adjoint(p2, v)


for name, fn in (("sequential", seq), ("two streams", conc)):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 5, "ms per fwd+adj")
