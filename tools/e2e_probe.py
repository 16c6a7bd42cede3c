"""Host-copy overlap probe: device-resident vs host-buffer calls on config 3."""
import time
import numpy as np
import torch
import paper_1809_10786_b200 as sgl
from paper_1809_10786_b200 import _native, workloads

w = workloads.config(3)
p = sgl.plan(w.B, w.points, q=16)
L = _native.lib()
pin = lambda a: (lambda t: (t.numpy().__setitem__(slice(None), a), t.numpy())[1])(
    torch.empty(a.shape, dtype=torch.complex128, pin_memory=True))
c_h, v_h = pin(w.coeffs[0] if w.coeffs.ndim == 2 else w.coeffs), pin(w.values)
fo, ao = pin(np.zeros(w.M, complex)), pin(np.zeros(p.count, complex))
c_d, v_d = torch.as_tensor(c_h).cuda(), torch.as_tensor(v_h).cuda()


def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / n


dev = lambda: (sgl.forward(p, c_d), sgl.adjoint(p, v_d))
sep = lambda: (_native.check(L.sgl_forward(p._handle, c_h.ctypes.data, 1, fo.ctypes.data, None)),
               _native.check(L.sgl_adjoint(p._handle, v_h.ctypes.data, ao.ctypes.data, None)))
fus = lambda: _native.check(L.sgl_forward_adjoint(p._handle, c_h.ctypes.data, fo.ctypes.data, v_h.ctypes.data,
                                                  ao.ctypes.data, None))
h2d = lambda: v_d.copy_(torch.from_numpy(v_h), non_blocking=True)
print({"device_ms": t(dev), "separate_host_ms": t(sep), "fused_host_ms": t(fus), "h2d_160MB_ms": t(h2d)})
fo_d, ao_d = torch.empty_like(v_d), torch.empty(p.count, dtype=torch.complex128, device="cuda")
F = lambda c, fo_, v, ao_: (lambda: _native.check(L.sgl_forward_adjoint(p._handle, c, fo_, v, ao_, None)))
print({"fused_dev_dev": t(F(c_d.data_ptr(), fo_d.data_ptr(), v_d.data_ptr(), ao_d.data_ptr())),
       "fused_hostin_devout": t(F(c_h.ctypes.data, fo_d.data_ptr(), v_h.ctypes.data, ao_d.data_ptr())),
       "fused_devin_hostout": t(F(c_d.data_ptr(), fo.ctypes.data, v_d.data_ptr(), ao.ctypes.data)),
       "fused_host_host": t(fus)})
