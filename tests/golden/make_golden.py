"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container, where the read-only reference is importable:

    python tests/golden/make_golden.py [--skip-big]

It imports `sglnufft` from /root/reference/pkg/src, builds each input with
the reference's own generators (draw order of SURVEY.md 8(d)), runs the
reference `plan / forward / adjoint` (numba backend, defaults sigma=2,
q=16 unless stated) and stores inputs + outputs as compressed .npz
fixtures next to this script.  Nothing on the GPU box reads
/root/reference; the tests only read these fixtures.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import sglnufft  # noqa: E402
    return sglnufft


def _vals(rng, M):
    re = rng.uniform(-1.0, 1.0, M)
    im = rng.uniform(-1.0, 1.0, M)
    return re + 1j * im


def small_cases(ref):
    """Small shapes covering sigma escalation, compact_k1, small q, and nodes
    on grid lines / the r = rho and r = 0 boundaries / the poles."""
    out = {}
    specs = [
        # name, B, M, q, compact, radius, seed
        ("b1_q4", 1, 7, 4, False, 2.0, 101),
        ("b2_q8", 2, 10, 8, False, 2.0, 102),
        ("b4_q8", 4, 30, 8, False, 2.0, 103),
        ("b5_q10", 5, 40, 10, False, 2.5, 104),
        ("b8_q16", 8, 200, 16, False, 3.0, 105),
        ("b6_q6_compact", 6, 100, 6, True, 4.0, 106),
        ("b12_q12", 12, 300, 12, False, 3.5, 107),
    ]
    for name, B, M, q, compact, rad, seed in specs:
        rng = np.random.Generator(np.random.PCG64(seed))
        c = ref.gen_coeffs(B, rng)
        pts = ref.gen_points_ball(M, rad, rng)
        v = _vals(rng, M)
        p = ref.plan(B, pts, q=q, compact_k1=compact)
        out[name] = dict(B=B, q=q, compact=compact, points=pts, coeffs=c, values=v, rho=p.rho,
                         fwd=ref.forward(p, c), adj=ref.adjoint(p, v))
    # special nodes: r = rho (x0 = 0 exactly), r = 0 (x0 = pi), poles, phi = 0,
    # and Cartesian-grid nodes whose warped coordinates fall on grid lines.
    for name, B, q in [("edges_b8_q16", 8, 16), ("edges_b3_q2", 3, 2), ("edges_b4_q5", 4, 5)]:
        rng = np.random.Generator(np.random.PCG64(200 + B))
        c = ref.gen_coeffs(B, rng)
        special = np.array([
            [2.0, 0.0, 0.0], [2.0, np.pi, 0.0], [0.0, 0.0, 0.0], [0.0, 1.0, 2.0],
            [1.0, np.pi / 2, 0.0], [2.0, np.pi / 2, np.pi], [1.5, np.pi / 4, 3 * np.pi / 2],
            [1.0, np.pi / 2, 2 * np.pi - 1e-17], [0.5, 0.0, 1.0],
        ])
        grid = ref.gen_grid(6, 1.0)
        pts = np.concatenate([special, grid, ref.gen_points_ball(40, 2.0, rng)])
        v = _vals(rng, pts.shape[0])
        p = ref.plan(B, pts, q=q)
        out[name] = dict(B=B, q=q, compact=False, points=pts, coeffs=c, values=v, rho=p.rho,
                         fwd=ref.forward(p, c), adj=ref.adjoint(p, v))
    return out


def cfg_cases(ref, skip_big):
    out = {}
    # config 1 at full size: B=16, M=20000 N(0, I/2), seed 0 (forward; adjoint too)
    rng = np.random.Generator(np.random.PCG64(0))
    B = 16
    c = ref.gen_coeffs(B, rng)
    from sglnufft.generate import cartesian_to_spherical
    pts = cartesian_to_spherical(rng.normal(0.0, np.sqrt(0.5), (20_000, 3)))
    v = _vals(rng, 20_000)
    t = time.time()
    p = ref.plan(B, pts)
    out["cfg1"] = dict(B=B, q=16, compact=False, points=pts, coeffs=c, values=v, rho=p.rho,
                       fwd=ref.forward(p, c), adj=ref.adjoint(p, v))
    print(f"cfg1 {time.time() - t:.1f}s", flush=True)

    # config 2 shape: B=32, gen_grid(100, 4.0); 2000-node seeded subset, rho pinned
    rng = np.random.Generator(np.random.PCG64(0))
    B = 32
    c = ref.gen_coeffs(B, rng)
    full = ref.gen_grid(100, 4.0)
    vfull = _vals(rng, full.shape[0])
    rho = float(np.max(full[:, 0]))
    sel = np.sort(np.random.Generator(np.random.PCG64(1)).choice(full.shape[0], 2000, replace=False))
    t = time.time()
    p = ref.plan(B, full[sel], rho=rho)
    out["cfg2_sub2000"] = dict(B=B, q=16, compact=False, points=full[sel], coeffs=c, values=vfull[sel],
                               rho=rho, sel=sel, fwd=ref.forward(p, c), adj=ref.adjoint(p, vfull[sel]))
    print(f"cfg2 {time.time() - t:.1f}s", flush=True)

    # config 3 shape: B=64, c / n, ball radius 16, M = 1e7 -> 600-node subset
    rng = np.random.Generator(np.random.PCG64(0))
    B = 64
    c = ref.gen_coeffs(B, rng)
    nmu = ref.indexing.mu_to_nlm_array(B)[:, 0]
    c = c / nmu
    Mf = 10_000_000
    full = ref.gen_points_ball(Mf, 16.0, rng)
    vfull = _vals(rng, Mf)
    rho = float(np.max(full[:, 0]))
    sel = np.sort(np.random.Generator(np.random.PCG64(1)).choice(Mf, 600, replace=False))
    t = time.time()
    p = ref.plan(B, full[sel], rho=rho)
    out["cfg3_sub600"] = dict(B=B, q=16, compact=False, points=full[sel], coeffs=c, values=vfull[sel],
                              rho=rho, sel=sel, fwd=ref.forward(p, c), adj=ref.adjoint(p, vfull[sel]),
                              head=full[:8], vhead=vfull[:8])
    print(f"cfg3 {time.time() - t:.1f}s", flush=True)
    del full, vfull

    # config 5 shape: B=48 (sigma_eff = 8/3), 64 vectors, 2e6 N(0, I/2) nodes -> 400-node subset, 2 vectors
    rng = np.random.Generator(np.random.PCG64(0))
    B = 48
    cs = np.stack([ref.gen_coeffs(B, rng) for _ in range(64)])
    Mf = 2_000_000
    full = cartesian_to_spherical(rng.normal(0.0, np.sqrt(0.5), (Mf, 3)))
    rho = float(np.max(full[:, 0]))
    sel = np.sort(np.random.Generator(np.random.PCG64(1)).choice(Mf, 400, replace=False))
    t = time.time()
    p = ref.plan(B, full[sel], rho=rho)
    fw = np.stack([ref.forward(p, cs[k]) for k in (0, 63)])
    out["cfg5_sub400"] = dict(B=B, q=16, compact=False, points=full[sel], coeffs=cs[[0, 63]], rho=rho,
                              sel=sel, fwd=fw, head=full[:8])
    print(f"cfg5 {time.time() - t:.1f}s", flush=True)
    del full

    if not skip_big:
        # config 4 shape: B=128, adjoint only (the reference forward is NaN here);
        # 120-node subset of the 50/50 mixture; rho pinned to the full 1e8 set.
        rng = np.random.Generator(np.random.PCG64(0))
        B = 128
        _ = ref.gen_coeffs(B, rng)
        Mf = 100_000_000
        h = Mf // 2
        a = cartesian_to_spherical(rng.normal(0.0, np.sqrt(0.5), (h, 3)))
        b = ref.gen_points_ball(Mf - h, 22.0, rng)
        perm = rng.permutation(Mf)
        vfull = _vals(rng, Mf)
        rho = float(max(a[:, 0].max(), b[:, 0].max()))
        sel = np.sort(np.random.Generator(np.random.PCG64(1)).choice(Mf, 120, replace=False))
        src = perm[sel]
        pts = np.where((src < h)[:, None], a[np.minimum(src, h - 1)], b[np.maximum(src - h, 0)])
        vals = vfull[sel]
        del a, b, vfull, perm
        t = time.time()
        p = ref.plan(B, pts, rho=rho)
        out["cfg4_sub120"] = dict(B=B, q=16, compact=False, points=pts, values=vals, rho=rho, sel=sel,
                                  adj=ref.adjoint(p, vals))
        print(f"cfg4 {time.time() - t:.1f}s", flush=True)
    return out


def scale_cases(ref):
    """Round-2 parity subsets at the sizes SURVEY 8(d) asks for: config 3 on a
    20k-node subset (forward + adjoint), config 2 on a 20k-node subset, and
    config 5 with ALL 64 vectors on a 2k-node subset plus 4 vectors on a
    20k-node subset.  rho is pinned to the full node set's.  Coefficients of
    configs 3 and 5 are not stored (39 MB for config 5): the tests regenerate
    them with the package's restated generators and check them against the
    stored fingerprints (`c_head`, `c_sum`) first."""
    from sglnufft.generate import cartesian_to_spherical
    out = {}
    # config 3: B=64, c / n, ball radius 16, M = 1e7 -> 20k-node subset
    rng = np.random.Generator(np.random.PCG64(0))
    B = 64
    c = ref.gen_coeffs(B, rng) / ref.indexing.mu_to_nlm_array(B)[:, 0]
    Mf = 10_000_000
    full = ref.gen_points_ball(Mf, 16.0, rng)
    vfull = _vals(rng, Mf)
    rho = float(np.max(full[:, 0]))
    sel = np.sort(np.random.Generator(np.random.PCG64(2)).choice(Mf, 20_000, replace=False))
    t = time.time()
    p = ref.plan(B, full[sel], rho=rho)
    out["cfg3_sub20k"] = dict(B=B, q=16, compact=False, points=full[sel], values=vfull[sel], rho=rho, sel=sel,
                              c_head=c[:64], c_sum=np.array([c.sum(), np.abs(c).sum()]),
                              fwd=ref.forward(p, c), adj=ref.adjoint(p, vfull[sel]))
    print(f"cfg3_sub20k {time.time() - t:.1f}s", flush=True)
    del full, vfull

    # config 2: B=32, gen_grid(100, 4.0) -> 20k-node subset
    rng = np.random.Generator(np.random.PCG64(0))
    B = 32
    c = ref.gen_coeffs(B, rng)
    full = ref.gen_grid(100, 4.0)
    vfull = _vals(rng, full.shape[0])
    rho = float(np.max(full[:, 0]))
    sel = np.sort(np.random.Generator(np.random.PCG64(2)).choice(full.shape[0], 20_000, replace=False))
    t = time.time()
    p = ref.plan(B, full[sel], rho=rho)
    out["cfg2_sub20k"] = dict(B=B, q=16, compact=False, points=full[sel], coeffs=c, values=vfull[sel], rho=rho,
                              sel=sel, fwd=ref.forward(p, c), adj=ref.adjoint(p, vfull[sel]))
    print(f"cfg2_sub20k {time.time() - t:.1f}s", flush=True)

    # config 5: B=48, 64 vectors, 2e6 N(0, I/2) nodes: all 64 vectors on 2k
    # nodes, vectors 0, 21, 42, 63 on 20k nodes
    rng = np.random.Generator(np.random.PCG64(0))
    B = 48
    cs = np.stack([ref.gen_coeffs(B, rng) for _ in range(64)])
    Mf = 2_000_000
    full = cartesian_to_spherical(rng.normal(0.0, np.sqrt(0.5), (Mf, 3)))
    rho = float(np.max(full[:, 0]))
    fp = dict(c_head=cs[:, :16], c_sum=np.stack([cs.sum(axis=1), np.abs(cs).sum(axis=1)], axis=1))
    sel = np.sort(np.random.Generator(np.random.PCG64(2)).choice(Mf, 2_000, replace=False))
    t = time.time()
    p = ref.plan(B, full[sel], rho=rho)
    fw = np.stack([ref.forward(p, cs[k]) for k in range(64)])
    out["cfg5_sub2k_all64"] = dict(B=B, q=16, compact=False, points=full[sel], rho=rho, sel=sel, fwd=fw,
                                   vectors=np.arange(64), **fp)
    print(f"cfg5_sub2k_all64 {time.time() - t:.1f}s", flush=True)
    sel = np.sort(np.random.Generator(np.random.PCG64(3)).choice(Mf, 20_000, replace=False))
    vec = np.array([0, 21, 42, 63])
    t = time.time()
    p = ref.plan(B, full[sel], rho=rho)
    fw = np.stack([ref.forward(p, cs[k]) for k in vec])
    out["cfg5_sub20k_4v"] = dict(B=B, q=16, compact=False, points=full[sel], rho=rho, sel=sel, fwd=fw,
                                 vectors=vec, **fp)
    print(f"cfg5_sub20k_4v {time.time() - t:.1f}s", flush=True)
    return out


def invert_cases(ref):
    """The CG inverse (solvers.py:204-277) on small systems: CGNR and CGNE."""
    out = {}
    for name, B, M, rad, seed, it in [("inv_cgnr_b4", 4, 200, 2.5, 301, 60), ("inv_cgne_b6", 6, 60, 2.0, 302, 40)]:
        rng = np.random.Generator(np.random.PCG64(seed))
        c = ref.gen_coeffs(B, rng)
        pts = ref.gen_points_ball(M, rad, rng)
        vals = ref.forward(ref.plan(B, pts), c)
        rep = ref.invert(pts, vals, B, max_iter=it, tol=1e-12, true_coeffs=c)
        out[name] = dict(B=B, q=16, compact=False, points=pts, coeffs=c, values=vals,
                         solution=rep.solution, iterations=rep.iterations, converged=rep.converged,
                         residual_history=np.array(rep.residual_history),
                         abs_error_history=np.array(rep.abs_error_history))
    # midpoint seed (solvers.py:166-191) on Cartesian-grid samples + CGNR from it
    B, kappa, N = 4, 1.5, 8
    pts = ref.gen_grid(N, kappa)
    rng = np.random.Generator(np.random.PCG64(303))
    c = ref.gen_coeffs(B, rng)
    vals = ref.forward(ref.plan(B, pts), c)
    from sglnufft.solvers import midpoint_initial_guess
    x0 = midpoint_initial_guess(vals, pts, B, kappa, N)
    rep = ref.invert(pts, vals, B, x0_mode="midpoint", kappa=kappa, grid_n=N, max_iter=30, tol=1e-12)
    out["inv_mid_b4"] = dict(B=B, q=16, compact=False, points=pts, coeffs=c, values=vals, kappa=kappa, grid_n=N,
                             x0=x0, solution=rep.solution, iterations=rep.iterations, converged=rep.converged,
                             residual_history=np.array(rep.residual_history))
    return out


def direct_cases(ref):
    """The reference's direct sums evaluate_direct / evaluate_direct_adjoint
    (transform.py:95-139) at small B, including r = 0, the poles and phi = 0."""
    out = {}
    special = np.array([[0.0, 0.0, 0.0], [0.0, 1.0, 2.0], [1.0, 0.0, 0.3], [1.2, np.pi, 5.0],
                        [2.0, np.pi / 2, 0.0], [0.7, 1e-9, 2 * np.pi - 1e-12], [2.5, 2.0, np.pi]])
    for name, B, M, rad, seed in [("direct_b1", 1, 5, 1.0, 401), ("direct_b7", 7, 60, 2.0, 402),
                                  ("direct_b16", 16, 200, 3.5, 403), ("direct_b24", 24, 120, 4.0, 404)]:
        rng = np.random.Generator(np.random.PCG64(seed))
        c = ref.gen_coeffs(B, rng)
        pts = np.concatenate([special, ref.gen_points_ball(M, rad, rng)])
        v = _vals(rng, pts.shape[0])
        out[name] = dict(B=B, points=pts, coeffs=c, values=v, fwd=ref.transform.evaluate_direct(c, B, pts),
                         adj=ref.transform.evaluate_direct_adjoint(v, B, pts))
    return out


def nfft_cases(ref):
    """The reference NFFT layer (nfft.py): nfft_plan / nfft_execute /
    nfft_adjoint_execute and the exact ndft / ndft_adjoint, d = 3, nodes
    outside [0, 2 pi) included (reduced by the plan)."""
    out = {}
    specs = [("nfft_a", (8, 10, 6), 2, 6, 300, 501), ("nfft_b", (16, 16, 16), 2, 16, 500, 502),
             ("nfft_c", (12, 8, 20), 3, 10, 400, 503), ("nfft_d", (32, 32, 16), 2, 16, 2000, 504),
             ("nfft_e", (10, 12, 8), (2, 4, 3), 8, 250, 506)]
    for name, n, sigma, q, M, seed in specs:
        rng = np.random.Generator(np.random.PCG64(seed))
        nodes = rng.uniform(-1.0, 2 * np.pi + 1.0, (M, 3))
        nodes[:5] = [[0, 0, 0], [2 * np.pi, 0, -1e-17], [np.pi, np.pi / 2, 3.0], [-np.pi, 1e-3, 6.2], [1, 2, 3]]
        f = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        v = _vals(rng, M)
        p = ref.nfft.nfft_plan(3, n, sigma, q, nodes)
        d = dict(n=np.array(n), sigma=np.array(sigma), q=q, nodes=nodes, coeffs=f, values=v,
                 fwd=ref.nfft.nfft_execute(p, f), adj=ref.nfft.nfft_adjoint_execute(p, v))
        if M <= 400:
            d["ndft"] = ref.nfft.ndft(3, n, f, nodes)
            d["ndft_adj"] = ref.nfft.ndft_adjoint(3, n, v, nodes)
        out[name] = d
    for name, d, n, sigma, q, M, seed in [("nfft_d1", 1, (16,), 2, 8, 120, 507),
                                          ("nfft_d2", 2, (12, 10), (2, 3), 6, 200, 508),
                                          ("nfft_d2b", 2, (32, 16), 2, 16, 300, 509)]:
        rng = np.random.Generator(np.random.PCG64(seed))
        nodes = rng.uniform(-1.0, 2 * np.pi + 1.0, (M, d))
        f = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        v = _vals(rng, M)
        p = ref.nfft.nfft_plan(d, n, sigma, q, nodes)
        out[name] = dict(d=d, n=np.array(n), sigma=np.array(sigma), q=q, nodes=nodes, coeffs=f, values=v,
                         fwd=ref.nfft.nfft_execute(p, f), adj=ref.nfft.nfft_adjoint_execute(p, v),
                         ndft=ref.nfft.ndft(d, n, f, nodes), ndft_adj=ref.nfft.ndft_adjoint(d, n, v, nodes))
    rng = np.random.Generator(np.random.PCG64(505))
    pts = ref.gen_points_ball(20, 3.0, rng)
    idx = np.array([(1, 0, 0), (3, 2, -1), (5, 4, 3), (8, 3, 0), (6, 5, -5)])
    basis = np.stack([ref.special.sgl_basis_eval(tuple(int(v) for v in t), pts) for t in idx])
    out["nfft_index"] = dict(nlm=ref.indexing.mu_to_nlm_array(10), basis_idx=idx, basis_pts=pts, basis=basis)
    return out


def precise_cases(ref):
    """forward / adjoint with precise=True (80-bit recurrences, recurrences.py:13)."""
    out = {}
    for name, B, M, q, rad, seed in [("precise_b8", 8, 200, 16, 3.0, 601), ("precise_b24", 24, 300, 12, 5.0, 602)]:
        rng = np.random.Generator(np.random.PCG64(seed))
        c = ref.gen_coeffs(B, rng)
        pts = ref.gen_points_ball(M, rad, rng)
        v = _vals(rng, M)
        p = ref.plan(B, pts, q=q)
        out[name] = dict(B=B, q=q, compact=False, points=pts, coeffs=c, values=v, rho=p.rho,
                         fwd=ref.forward(p, c, precise=True), adj=ref.adjoint(p, v, precise=True),
                         fwd_double=ref.forward(p, c), adj_double=ref.adjoint(p, v))
    return out


def csv_cases(ref):
    """Files written by the reference CLI (cli.py) itself: generators and the
    three transform methods on a small problem (tests/golden/csv/)."""
    import shutil
    import tempfile
    from sglnufft import cli
    d = os.path.join(HERE, "csv")
    os.makedirs(d, exist_ok=True)
    tmp = tempfile.mkdtemp()
    runs = [
        ["gen-coeffs", "-B", "5", "--seed", "7", "--out", "c_b5.csv"],
        ["gen-points", "-M", "40", "--kappa", "2.5", "--seed", "3", "--out", "p_m40.csv"],
        ["gen-grid", "-N", "4", "--kappa", "1.5", "--out", "g_n4.csv"],
        ["forward", "--coeffs", "c_b5.csv", "--points", "p_m40.csv", "--method", "naive", "--out", "f_naive.csv"],
        ["forward", "--coeffs", "c_b5.csv", "--points", "p_m40.csv", "-q", "8", "--out", "f_fast.csv"],
        ["forward", "--coeffs", "c_b5.csv", "--points", "p_m40.csv", "--method", "fast-exact",
         "--out", "f_exact.csv"],
        ["adjoint", "--values", "f_naive.csv", "--points", "p_m40.csv", "-B", "5", "--method", "naive",
         "--out", "a_naive.csv"],
        ["adjoint", "--values", "f_naive.csv", "--points", "p_m40.csv", "-B", "5", "-q", "8", "--out", "a_fast.csv"],
        ["invert", "--values", "f_naive.csv", "--points", "p_m40.csv", "-B", "3", "--max-iter", "50",
         "--out", "inv_b3.csv"],
        ["experiment", "error-vs-q", "-B", "5", "-M", "80", "--kappa", "3.0", "--q-list", "2,4,8,12,16",
         "--repetitions", "3", "--seed", "11", "--out", "exp_q.csv"],
        ["experiment", "error-vs-radius", "-B", "4", "-M", "60", "--kappa-list", "0.5,2,4", "-q", "10",
         "--repetitions", "2", "--seed", "12", "--out", "exp_radius.csv"],
        ["experiment", "error-vs-bandwidth", "--bandwidth-list", "3,6", "-M", "50", "--kappa", "2.5", "-q", "8",
         "--repetitions", "2", "--seed", "13", "--exact-control", "--out", "exp_bw.csv"],
        ["experiment", "inverse-convergence", "-B", "3", "-q", "8", "--grid-n-list", "6", "--kappa", "1.5",
         "--max-iter", "12", "--seed", "14", "--out", "exp_inv.csv"],
    ]
    cwd = os.getcwd()
    os.chdir(tmp)
    try:
        for argv in runs:
            rc = cli.main(argv)
            assert rc == 0, argv
        for f in sorted(os.listdir(tmp)):
            shutil.copy(os.path.join(tmp, f), os.path.join(d, f))
            print("wrote", os.path.join(d, f))
    finally:
        os.chdir(cwd)
        shutil.rmtree(tmp)
    with open(os.path.join(d, "RUNS.txt"), "w") as fh:
        fh.write("\n".join(" ".join(r) for r in runs) + "\n")
    return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-big", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    ref = _ref()
    cases = {}
    if args.only in ("", "small"):
        cases.update(small_cases(ref))
    if args.only in ("", "cfg"):
        cases.update(cfg_cases(ref, args.skip_big))
    if args.only in ("", "scale"):
        cases.update(scale_cases(ref))
    if args.only in ("", "invert"):
        cases.update(invert_cases(ref))
    if args.only in ("", "direct"):
        cases.update(direct_cases(ref))
    if args.only in ("", "csv"):
        csv_cases(ref)
    if args.only in ("", "nfft"):
        cases.update(nfft_cases(ref))
    if args.only in ("", "precise"):
        cases.update(precise_cases(ref))
    for name, d in cases.items():
        path = os.path.join(HERE, f"ref_{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in d.items()})
        print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
