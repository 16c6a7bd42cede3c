"""Parity of the CUDA path (through the C ABI) with the reference.

Goldens are outputs of the reference package itself (tests/golden/).  The bar
is rel-linf = max|x - ref| / max|ref| <= 1e-10 (BASELINE north star; the
reference's own idiom, test_transform.py:223, 303); the measured CPU rounding
floor is 1e-15 .. 3e-14.
"""
import numpy as np
import pytest

from conftest import SMALL, load_golden

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(x, ref):
    x, ref = np.asarray(x), np.asarray(ref)
    return float(np.max(np.abs(x - ref)) / np.max(np.abs(ref)))


@pytest.fixture(scope="module")
def sgl():
    import paper_1809_10786_b200 as m
    from paper_1809_10786_b200 import _native
    assert _native.device_count() >= 1, "no CUDA device: the -m gpu suite needs a B200"
    return m


def _plan(sgl, g, **kw):
    return sgl.plan(int(g["B"]), g["points"], q=int(g["q"]), rho=float(g["rho"]),
                    compact_k1=bool(g["compact"]), **kw)


@pytest.mark.parametrize("backend", ["auto", "tiled", "generic"])
@pytest.mark.parametrize("name", SMALL + ["cfg1", "cfg2_sub2000", "cfg3_sub600", "cfg5_sub400"])
def test_forward_adjoint_match_reference(sgl, name, backend):
    # auto: int8 tensor-core gather (q <= 16); tiled: FP64 DMMA kernels both ways
    g = load_golden(name)
    if backend == "generic" and name.startswith("cfg") and name != "cfg1":
        pytest.skip("generic kernels cross-checked on the small and cfg1 shapes")
    p = _plan(sgl, g, backend=backend)
    assert p.rho == float(g["rho"])
    f = sgl.forward(p, g["coeffs"])
    assert f.shape == g["fwd"].shape
    assert rel(f, g["fwd"]) <= TOL, rel(f, g["fwd"])
    if "adj" in g:
        a = sgl.adjoint(p, g["values"])
        assert rel(a, g["adj"]) <= TOL, rel(a, g["adj"])


# Config 4 (B = 128, rho = 22) is ill-conditioned in FP64: the adjoint entries
# span 1 .. 1e95 and rounding is amplified by the radial functions.  Against
# the extended-precision truth (tests/golden/ref_cfg4_truth.npz,
# test_parity_scale_gpu.py) the reference's own fast adjoint is 2.56e-9 off
# and ours 1.22e-9 (basal matrices built in extended precision); two values
# that far from the truth can differ from each other by up to their sum, so
# the bar against the reference's output is 2 x its own error.
TOL_CFG4 = 2 * 2.56e-9


def test_config4_adjoint_matches_reference(sgl):
    # B = 128, rho pinned to the full 1e8-node set; the reference forward is NaN here
    g = load_golden("cfg4_sub120")
    p = sgl.plan(128, g["points"], rho=float(g["rho"]))
    a = sgl.adjoint(p, g["values"])
    assert np.all(np.isfinite(a))
    assert rel(a, g["adj"]) <= TOL_CFG4, rel(a, g["adj"])
    # our forward stays finite where the reference overflows (transform.py:226)
    f = sgl.forward(p, np.ones(p.count, dtype=complex))
    assert np.all(np.isfinite(f))


@pytest.mark.parametrize("name", ["b8_q16", "b5_q10", "edges_b8_q16", "cfg1"])
def test_tiled_and_generic_kernels_agree(sgl, name):
    # the reference's TestBackends pattern (test_nfft.py:213-225)
    g = load_golden(name)
    pa, pb = _plan(sgl, g, backend="tiled"), _plan(sgl, g, backend="generic")
    assert pa.stats["n_tiles"] > 0 and pb.stats["generic"]
    assert rel(sgl.forward(pa, g["coeffs"]), sgl.forward(pb, g["coeffs"])) <= 1e-12
    assert rel(sgl.adjoint(pa, g["values"]), sgl.adjoint(pb, g["values"])) <= 1e-12


def test_grid_line_nodes_tiled(sgl):
    # a Cartesian lattice (config 2's generator) puts many nodes exactly on
    # grid lines of axes 1-2 (phi = k pi/2, theta = pi/2): they are tiled in
    # their own single-cell pencils; results equal the per-node kernels and
    # the oracle, and tiles stay full
    from oracle import sgl_oracle as o
    pts = sgl.gen_grid(20, 3.0)
    rng = np.random.default_rng(5)
    c = sgl.gen_coeffs(12, rng)
    v = rng.uniform(-1, 1, len(pts)) + 1j * rng.uniform(-1, 1, len(pts))
    pa, pb = sgl.plan(12, pts, backend="tiled"), sgl.plan(12, pts, backend="generic")
    fa, aa = sgl.forward(pa, c), sgl.adjoint(pa, v)
    assert rel(fa, sgl.forward(pb, c)) <= 1e-12 and rel(aa, sgl.adjoint(pb, v)) <= 1e-12
    op = o.oracle_plan(12, pts)
    assert rel(fa, o.oracle_forward(op, c)) <= TOL and rel(aa, o.oracle_adjoint(op, v)) <= TOL


@pytest.mark.parametrize("B,M,q,rad", [(5, 40, 10, 2.5), (8, 500, 16, 3.0), (16, 3000, 16, 4.0), (6, 200, 20, 2.0)])
def test_pairing(sgl, B, M, q, rad):
    # <y, F x> == <F^H y, x> (test_transform.py:305-315)
    rng = np.random.default_rng(32 + B)
    pts = sgl.gen_points_ball(M, rad, rng)
    p = sgl.plan(B, pts, q=q)
    x = sgl.gen_coeffs(B, rng)
    y = rng.normal(size=M) + 1j * rng.normal(size=M)
    fx = sgl.forward(p, x)
    lhs = np.vdot(y, fx)
    rhs = np.vdot(sgl.adjoint(p, y), x)
    # the reference's bound (1e-11 |x| |y|, written for B = 5, q = 10), plus the
    # same relative bound on the scale of <y, F x> for the larger operators
    # (B = 16, rho = 4: |F x| / |x| ~ 30); the default forward is the int8
    # gather (~1e-13 relative), the adjoint the FP64 scatter
    assert abs(lhs - rhs) <= 1e-11 * np.linalg.norm(y) * (np.linalg.norm(x) + np.linalg.norm(fx))


def test_linearity_zero_and_errors(sgl):
    rng = np.random.default_rng(22)
    B = 4
    pts = sgl.gen_points_ball(30, 2.0, rng)
    p = sgl.plan(B, pts, q=8)
    x, y = sgl.gen_coeffs(B, rng), sgl.gen_coeffs(B, rng)
    a, b = 1.3 - 0.2j, -0.7 + 1.1j
    lhs = sgl.forward(p, a * x + b * y)
    rhs = a * sgl.forward(p, x) + b * sgl.forward(p, y)
    assert rel(lhs, rhs) <= 1e-10
    assert np.all(sgl.adjoint(p, np.zeros(30)) == 0)
    assert np.all(sgl.forward(p, np.zeros(p.count)) == 0)
    with pytest.raises(ValueError):
        sgl.forward(p, np.zeros(p.count + 1))
    with pytest.raises(ValueError):
        sgl.adjoint(p, np.zeros(31))
    with pytest.raises(ValueError):
        sgl.plan(2, np.array([[2.1, 0, 0]]), q=4, rho=1.0)


@pytest.mark.parametrize("name", ["precise_b8", "precise_b24"])
def test_precise_matches_reference_precise(sgl, name):
    # precise=True: basal tables in x87 extended precision on a cached twin
    # plan; against the reference's own precise=True outputs
    # (default plans build their tables in extended precision: precise calls
    # run on the plan itself; FP64-table plans get a cached twin)
    g = load_golden(name)
    p = _plan(sgl, g)
    assert p.precise_tables
    f = sgl.forward(p, g["coeffs"], precise=True)
    a = sgl.adjoint(p, g["values"], precise=True)
    assert rel(f, g["fwd"]) <= TOL and rel(a, g["adj"]) <= TOL
    assert p._twin is None
    assert rel(sgl.forward(p, g["coeffs"]), g["fwd_double"]) <= TOL
    p64 = _plan(sgl, g, precise_tables=False)
    assert rel(sgl.forward(p64, g["coeffs"]), g["fwd_double"]) <= TOL
    f = sgl.forward(p64, g["coeffs"], precise=True)
    assert rel(f, g["fwd"]) <= TOL
    assert p64._twin is not None and p64._twin.precise_tables
    assert sgl.forward(p64, g["coeffs"], precise=True).shape == f.shape   # the twin is reused
    p64.close()
    assert p64._twin is None


def test_compact_grid_agrees(sgl):
    g = load_golden("b8_q16")
    full = _plan(sgl, g)
    comp = sgl.plan(8, g["points"], compact_k1=True)
    assert comp.nfft.grid_shape[1] == full.nfft.grid_shape[1] // 2
    assert rel(sgl.forward(comp, g["coeffs"]), sgl.forward(full, g["coeffs"])) <= 1e-10
    assert rel(sgl.adjoint(comp, g["values"]), sgl.adjoint(full, g["values"])) <= 1e-10


def test_batched_forward_matches_single(sgl):
    g = load_golden("cfg5_sub400")
    p = _plan(sgl, g)
    fb = sgl.forward(p, g["coeffs"])
    assert fb.shape == (2, 400)
    for k in range(2):
        assert rel(fb[k], g["fwd"][k]) <= TOL
        assert np.array_equal(fb[k], sgl.forward(p, g["coeffs"][k]))


def test_batched_forward_host_double_buffer(sgl):
    """K = 5 vectors into host memory: downloads overlap the next vector on a
    side stream with two alternating value buffers."""
    g = load_golden("cfg2_sub2000")
    p = _plan(sgl, g)
    rng = np.random.default_rng(7)
    C = np.stack([sgl.gen_coeffs(int(g["B"]), rng) for _ in range(5)])
    fb = sgl.forward(p, C)
    for k in range(5):
        assert np.array_equal(fb[k], sgl.forward(p, C[k]))


def test_torch_device_tensors(sgl):
    import torch
    g = load_golden("b12_q12")
    dev = torch.device("cuda", 0)
    pts = torch.as_tensor(g["points"], device=dev)
    p = sgl.plan(12, pts, q=12, rho=float(g["rho"]))
    f = sgl.forward(p, torch.as_tensor(g["coeffs"], device=dev))
    assert f.is_cuda and f.dtype == torch.complex128
    assert rel(f.cpu().numpy(), g["fwd"]) <= TOL
    a = sgl.adjoint(p, torch.as_tensor(g["values"], device=dev))
    assert rel(a.cpu().numpy(), g["adj"]) <= TOL


@pytest.mark.parametrize("name", ["b12_q12", "cfg2_sub2000"])
def test_forward_adjoint_fused_call(sgl, name):
    """sgl_forward_adjoint == separate forward + adjoint (host buffers:
    side-stream copies; device tensors: plain stream order).  The forward is
    bit-identical; the adjoint's RED accumulation order varies run to run, so
    it agrees to rounding."""
    import torch
    g = load_golden(name)
    p = _plan(sgl, g)
    c = g["coeffs"] if g["coeffs"].ndim == 1 else g["coeffs"][0]
    f, a = sgl.forward_adjoint(p, c, g["values"])
    assert np.array_equal(f, sgl.forward(p, c))
    assert rel(a, sgl.adjoint(p, g["values"])) <= 1e-13
    assert rel(a, g["adj"]) <= TOL
    for _ in range(3):   # repeated calls reuse the side stream and buffers
        f2, a2 = sgl.forward_adjoint(p, c, g["values"])
        assert np.array_equal(f2, f) and rel(a2, a) <= 1e-13
    dev = torch.device("cuda", 0)
    fd, ad = sgl.forward_adjoint(p, torch.as_tensor(c, device=dev), torch.as_tensor(g["values"], device=dev))
    assert np.array_equal(fd.cpu().numpy(), f) and rel(ad.cpu().numpy(), a) <= 1e-13
    with pytest.raises(ValueError):
        sgl.forward_adjoint(p, c[:-1], g["values"])
    e = sgl.plan(3, np.zeros((0, 3)), q=4)
    fe, ae = sgl.forward_adjoint(e, np.ones(14), np.zeros(0))
    assert fe.shape == (0,) and np.all(ae == 0)


def test_empty_and_single_node(sgl):
    p = sgl.plan(3, np.zeros((0, 3)), q=4)
    assert sgl.forward(p, np.ones(14)).shape == (0,)
    assert np.all(sgl.adjoint(p, np.zeros(0)) == 0)
    g = load_golden("edges_b3_q2")
    from oracle import sgl_oracle as o
    pts = g["points"][:1]
    p1 = sgl.plan(3, pts, q=2, rho=float(g["rho"]))
    op = o.oracle_plan(3, pts, q=2, rho=float(g["rho"]))
    assert rel(sgl.forward(p1, g["coeffs"]), o.oracle_forward(op, g["coeffs"])) <= TOL


def test_config3_full_size(sgl):
    """BASELINE config 3 at full M = 1e7: the forward is pointwise, so the
    golden subset must match entry for entry; the adjoint is linear, so the
    GPU adjoint over all nodes with values zeroed outside the subset must
    match the reference adjoint of the subset."""
    from paper_1809_10786_b200 import workloads
    g = load_golden("cfg3_sub600")
    w = workloads.config(3)
    p = sgl.plan(64, w.points)
    assert p.rho == float(g["rho"])
    f = sgl.forward(p, w.coeffs)
    assert rel(f[g["sel"]], g["fwd"]) <= TOL
    v = np.zeros(w.M, dtype=complex)
    v[g["sel"]] = g["values"]
    a = sgl.adjoint(p, v)
    assert rel(a, g["adj"]) <= TOL
    # full-size property: pairing over all 1e7 nodes, relative to the
    # Cauchy-Schwarz scale |F x| |y| (entries of F x reach 1e53 here)
    lhs = np.vdot(w.values, f)
    rhs = np.vdot(sgl.adjoint(p, w.values), w.coeffs)
    assert abs(lhs - rhs) <= 1e-11 * np.linalg.norm(f) * np.linalg.norm(w.values)


def test_config4_full_size_adjoint(sgl):
    """BASELINE config 4 at full size (B = 128, M = 1e8 nodes, one GPU): the
    adjoint over all nodes with values zeroed outside the golden subset must
    match the reference adjoint of the subset."""
    from paper_1809_10786_b200 import workloads
    g = load_golden("cfg4_sub120")
    w = workloads.config(4)
    assert w.rho == float(g["rho"])
    assert np.array_equal(w.points[g["sel"]], g["points"])
    p = sgl.plan(128, w.points)
    v = np.zeros(w.M, dtype=complex)
    v[g["sel"]] = g["values"]
    del w
    a = sgl.adjoint(p, v)
    assert np.all(np.isfinite(a))
    assert rel(a, g["adj"]) <= TOL_CFG4, rel(a, g["adj"])


# --- exact last stage (transform.py:393-394, 404-405): direct NDFT on device ---

@pytest.mark.parametrize("B", [1, 2, 4, 8])
def test_exact_stage_matches_direct_sums(sgl, B):
    # reference test_transform.py:215-223, with the direct sums of the oracle
    from oracle import sgl_oracle as o
    rng = np.random.default_rng(10 + B)
    c = sgl.gen_coeffs(B, rng)
    pts = sgl.gen_points_ball(25, 3.0, rng)
    p = sgl.plan(B, pts, exact_last_stage=True)
    assert p.exact and p.q is None and p.nfft is None
    ref = o.evaluate_direct(c, B, pts)
    assert rel(sgl.forward(p, c), ref) <= 1e-10


def test_exact_stage_adjoint_and_pairing(sgl):
    # reference test_transform.py:296-315
    from oracle import sgl_oracle as o
    rng = np.random.default_rng(31)
    B, m = 6, 50
    pts = sgl.gen_points_ball(m, 3.0, rng)
    v = rng.normal(size=m) + 1j * rng.normal(size=m)
    p = sgl.plan(B, pts, exact_last_stage=True)
    assert rel(sgl.adjoint(p, v), o.evaluate_direct_adjoint(v, B, pts)) <= 1e-9
    x = sgl.gen_coeffs(B, rng)
    lhs = np.vdot(v, sgl.forward(p, x))
    rhs = np.vdot(sgl.adjoint(p, v), x)
    assert abs(lhs - rhs) <= 1e-11 * np.linalg.norm(x) * np.linalg.norm(v)


def test_exact_compact_grid_agrees(sgl):
    # reference test_transform.py:265-272
    rng = np.random.default_rng(23)
    B = 4
    c = sgl.gen_coeffs(B, rng)
    pts = sgl.gen_points_ball(40, 2.5, rng)
    ref = sgl.forward(sgl.plan(B, pts, exact_last_stage=True), c)
    out = sgl.forward(sgl.plan(B, pts, exact_last_stage=True, compact_k1=True), c)
    assert rel(out, ref) <= 1e-11


def test_fast_vs_exact_stage_window_error(sgl):
    # the fast path deviates from the exact stage only by the window error,
    # which decays in q (test_transform.py:225-252)
    rng = np.random.default_rng(20)
    B = 8
    c = sgl.gen_coeffs(B, rng)
    pts = sgl.gen_points_ball(300, 5.0, rng)
    exact = sgl.forward(sgl.plan(B, pts, exact_last_stage=True), c)
    errs = {q: rel(sgl.forward(sgl.plan(B, pts, q=q), c), exact) for q in (4, 8, 12, 16)}
    assert errs[16] <= 1e-4 * errs[4] and errs[16] <= 1e-9


def test_plan_shared_across_threads(sgl):
    """Concurrent forward/adjoint calls on one plan from several host threads
    (the reference's plans are shareable, README.md:66-67)."""
    import threading
    g = load_golden("b12_q12")
    p = sgl.plan(12, g["points"], q=12, rho=float(g["rho"]))
    res, errs = {}, []

    def work(k):
        try:
            for _ in range(5):
                res[("f", k)] = sgl.forward(p, g["coeffs"])
                res[("a", k)] = sgl.adjoint(p, g["values"])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    for k in range(4):
        assert rel(res[("f", k)], g["fwd"]) <= TOL and rel(res[("a", k)], g["adj"]) <= TOL


def test_cuda_graph_capture(sgl):
    """forward / adjoint on device tensors can be captured into a CUDA graph
    and replayed (e.g. a CG loop); replays match eager calls."""
    import torch
    g = load_golden("b12_q12")
    dev = torch.device("cuda", 0)
    p = sgl.plan(12, g["points"], q=12, rho=float(g["rho"]))
    c = torch.as_tensor(g["coeffs"], device=dev)
    v = torch.as_tensor(g["values"], device=dev)
    f0, a0 = sgl.forward(p, c).clone(), sgl.adjoint(p, v).clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        sgl.forward(p, c)
        sgl.adjoint(p, v)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        fo = sgl.forward(p, c)
        ao = sgl.adjoint(p, v)
    c.mul_(2.0)   # replays read the captured buffers' current contents
    graph.replay()
    torch.cuda.synchronize()
    assert rel(fo.cpu().numpy(), 2.0 * f0.cpu().numpy()) <= 1e-13
    assert rel(ao.cpu().numpy(), a0.cpu().numpy()) <= 1e-13
    assert rel(fo.cpu().numpy(), 2.0 * g["fwd"]) <= TOL
