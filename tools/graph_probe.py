import torch, numpy as np, time
import paper_1809_10786_b200 as sgl
B, N, q = 8, 25, 15
pts = sgl.gen_grid(N, 3.0)
c = sgl.gen_coeffs(B, 1)
p = sgl.plan(B, pts, q=q)
cd = torch.as_tensor(c, device="cuda"); vd = torch.randn(len(pts), dtype=torch.complex128, device="cuda")
f0 = sgl.forward(p, cd); a0 = sgl.adjoint(p, vd)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        sgl.forward(p, cd); sgl.adjoint(p, vd)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g):
        fo = sgl.forward(p, cd)
        ao = sgl.adjoint(p, vd)
    g.replay(); torch.cuda.synchronize()
    print("graph ok", float((fo - f0).abs().max() / f0.abs().max()), float((ao - a0).abs().max() / a0.abs().max()))
    t0 = time.perf_counter()
    for _ in range(200): g.replay()
    torch.cuda.synchronize()
    print("replay ms/pair", (time.perf_counter() - t0) * 5)
except Exception as e:
    print("graph capture failed:", type(e).__name__, str(e)[:300])
