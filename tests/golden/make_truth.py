"""Extended-precision truth for the config-4 golden subset.

    python tests/golden/make_truth.py

Config 4 (B = 128, rho = 22) is ill-conditioned in FP64: the reference's own
two FP64 paths (fast adjoint, `transform.adjoint`, and direct sums,
`transform.evaluate_direct_adjoint`, transform.py:120-139) disagree by
~2.6e-9 on `ref_cfg4_sub120`.  This script computes the direct adjoint of
that subset in longdouble (`oracle/extended.py`), pins it with mpmath at 60
digits on the largest and on random entries, measures the reference's own
paths against it, and stores `tests/golden/ref_cfg4_truth.npz`:

    truth        complex128 rounding of the longdouble direct adjoint
    ref_fast_err rel-linf of the reference fast adjoint (the golden `adj`)
    ref_direct_err rel-linf of the reference FP64 direct sums
    mp_mus, mp_vals, mp_err  the mpmath spot check

Runs in the build container (imports the reference from /root/reference for
the FP64 direct sums; nothing on the GPU box reads it).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def rel(x, ref):
    return float(np.max(np.abs(np.asarray(x) - ref)) / np.max(np.abs(ref)))


def main():
    from oracle import extended as X
    g = dict(np.load(os.path.join(HERE, "ref_cfg4_sub120.npz")))
    B, pts, vals = int(g["B"]), g["points"], g["values"]
    t = time.time()
    truth_ld = X.direct_adjoint_ld(vals, B, pts)
    truth = truth_ld.astype(complex)
    print(f"longdouble direct adjoint: {time.time() - t:.1f} s", flush=True)
    rng = np.random.default_rng(0)
    top = np.argsort(-np.abs(truth))[:12]
    mus = np.concatenate([top, rng.choice(truth.size, 12, replace=False)])
    t = time.time()
    mp_vals = X.mp_direct_adjoint_entries(vals, B, pts, mus, dps=60)
    mp_err = np.abs(mp_vals - truth[mus]) / np.max(np.abs(truth))
    print(f"mpmath spot check ({len(mus)} entries, {time.time() - t:.1f} s): "
          f"max |mp - ld| / max|truth| = {mp_err.max():.2e}", flush=True)
    sys.path.insert(0, "/root/reference/pkg/src")
    import sglnufft as ref
    direct = ref.transform.evaluate_direct_adjoint(vals, B, pts)
    out = dict(truth=truth, mp_mus=mus, mp_vals=mp_vals, mp_err=mp_err,
               ref_fast_err=rel(g["adj"], truth), ref_direct_err=rel(direct, truth),
               ref_fast_vs_direct=rel(g["adj"], direct))
    for k in ("ref_fast_err", "ref_direct_err", "ref_fast_vs_direct"):
        print(k, out[k])
    np.savez_compressed(os.path.join(HERE, "ref_cfg4_truth.npz"), **{k: np.asarray(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
