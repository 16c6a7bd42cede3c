"""int8 gather vs FP64 gather on adversarial SGL spectra: coefficients only at
the highest radial / angular degrees (trig volume concentrated at the spectral
edge, where the deconvolution gain is largest), white raw-NFFT spectra."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_10786_b200 as sgl  # noqa: E402
from paper_1809_10786_b200 import indexing  # noqa: E402

rng = np.random.default_rng(0)
for B, rad in [(8, 3.0), (16, 4.0), (32, 6.0)]:
    pts = sgl.gen_points_ball(20000, rad, rng)
    p8, p64 = sgl.plan(B, pts), sgl.plan(B, pts, backend="tiled")
    nlm = indexing.mu_to_nlm_array(B) if hasattr(indexing, "mu_to_nlm_array") else None
    for kind in ("uniform", "top-n", "top-l", "top-m"):
        c = sgl.gen_coeffs(B, rng)
        if nlm is not None and kind != "uniform":
            n, l, m = nlm[:, 0], nlm[:, 1], nlm[:, 2]
            keep = {"top-n": n == B, "top-l": l == B - 1, "top-m": np.abs(m) == B - 1}[kind]
            c = np.where(keep, c, 0)
        f8, f64 = sgl.forward(p8, c), sgl.forward(p64, c)
        e = np.abs(f8 - f64).max() / np.abs(f64).max()
        print(f"B={B} {kind:8s}: i8 vs fp64 rel-linf {e:.2e}", flush=True)
