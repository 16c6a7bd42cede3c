import numpy as np, time, paper_1809_10786_b200 as sgl
import sys; sys.path.insert(0, "tests"); from conftest import load_golden  # noqa: E402
from oracle import sgl_oracle as o
rel=lambda x,r: float(np.max(np.abs(x-r))/np.max(np.abs(r)))
for n in ["direct_b1","direct_b7","direct_b16","direct_b24"]:
    g=load_golden(n); B=int(g["B"])
    print(n, rel(sgl.evaluate_direct(g["coeffs"],B,g["points"]),g["fwd"]), rel(sgl.evaluate_direct_adjoint(g["values"],B,g["points"]),g["adj"]))
for B,M in [(40,200),(64,40)]:
    rng=np.random.default_rng(B); c=sgl.gen_coeffs(B,rng); pts=sgl.gen_points_ball(M,6.0,rng); v=rng.uniform(-1,1,M)+1j*rng.uniform(-1,1,M)
    print(B, rel(sgl.evaluate_direct(c,B,pts),o.evaluate_direct(c,B,pts)), rel(sgl.evaluate_direct_adjoint(v,B,pts),o.evaluate_direct_adjoint(v,B,pts)))
g=load_golden("cfg3_sub600"); B=64
pts,c,v=g["points"],g["coeffs"],g["values"]
f=sgl.evaluate_direct(c,B,pts); a=sgl.evaluate_direct_adjoint(v,B,pts)
p=sgl.plan(B,pts,rho=float(g["rho"]))
print("fast vs direct", rel(sgl.forward(p,c),f), rel(sgl.adjoint(p,v),a), "golden fwd vs direct", rel(g["fwd"],f))
import torch
for M in [10000, 100000]:
    rng=np.random.default_rng(1); P=sgl.gen_points_ball(M,16.0,rng); vv=rng.uniform(-1,1,M)+0j
    sgl.evaluate_direct(c,B,P[:10]); torch.cuda.synchronize()
    t=time.time(); sgl.evaluate_direct(c,B,P); t1=time.time()-t
    t=time.time(); sgl.evaluate_direct_adjoint(vv,B,P); t2=time.time()-t
    print("B=64 M",M,"fwd s",t1,"adj s",t2)
