"""NFSGLFT benchmark: nodes/sec of forward + adjoint at BASELINE config 3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3] [--points M] [--scaling strong|weak]
                    [--partition auto|coeffs|grid]

A step is one forward (coefficients -> values at all M nodes) plus one adjoint
(values -> coefficients) on a fixed plan: BASELINE.json's headline metric
"NFSGLFT nodes/sec fwd+adj at B=64" on config 3 (B=64, M=1e7 nodes uniform in
the radius-16 ball, complex128).  Inputs are the seeded synthetic inputs of
SURVEY 8(d) (no public dataset exists for this path).

N > 1 (torchrun, one rank per GPU), default --scaling strong: every rank
builds the SAME config (seed 0, same coefficients), takes its node shard
(--shard theta: an equal-count band in the polar angle, full node density;
contiguous / radial: distributed.shard_indices), rho is the all-reduce max
over the shards (= the full set's); value = M_total / the slowest rank's
step time.
The adjoint's exchange is the partition `distributed.partition_model` picks
(--partition overrides): the coefficient all-reduce or the north star's grid
reduce-scatter + slab FFT.  --scaling weak: each rank its own M-node set.

--impl reference times the reference itself: the unmodified `sglnufft`
package (numba, as shipped: serial window loops, single-threaded pocketfft)
installed in baseline/_ref, JIT warm-up excluded as the reference's own
runners do (experiments.py:240-243); per step two rho-pinned node samples
give T_fixed + M t_node, extrapolated to M and flagged as such.
The 16-thread oracle port (oracle/) is reported beside it (`cpu_port`), and
replaces it when the reference cannot be imported.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1   # measured: DMMA m8n8k4 loop, profiles/fp64_peak_r01.txt (MEASURED_PEAKS.json has no FP64 entry)
INT8_PEAK_TOPS = 4550.0   # measured: tcgen05.mma kind::i8 M=128 N=256 loop, profiles/i8_mma_rate_r01.txt
# int8 gather: per K-step 21 digit pairs x (M = 128 nodes) x (N = 80 (b, re|im)) x (K = 32) MACs
I8_OPS_PER_KSTEP = 2.0 * 21 * 128 * 80 * 32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--points", type=int, default=None, help="override the node count per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-sample", type=int, default=4000)
    ap.add_argument("--direction", default=None, choices=["both", "fwd", "adj"],
                    help="default: the config's own (3: both, 4: adj, 5: batched fwd)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--partition", default="auto", choices=["auto", "coeffs", "grid"])
    ap.add_argument("--shard", default="theta", choices=["theta", "contiguous", "radial"],
                    help="strong scaling: how the config's nodes are split over the ranks")
    ap.add_argument("--no-stock", action="store_true", help="skip timing the stock reference package")
    ap.add_argument("--backend", default="auto", choices=["auto", "tiled", "i8"],
                    help="window engines (experiments; the default is the library's own choice)")
    ap.add_argument("--deterministic", action="store_true",
                    help="bitwise reproducible adjoint (fixed-point grid reductions, SGL_FLAG_DETERMINISTIC)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t_end = time.time() + 1.0   # short timed regions: wait for the first sample (<= 1 s)
        while not any(r and r[0].replace(".", "").isdigit() for r in self.rows) and time.time() < t_end:
            time.sleep(0.02)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def metric_name(cfg: int, direction: str, B: int, K: int) -> str:
    """BASELINE.json's metric for its headline config; the same wording for
    the other configs (their parity-bench lines)."""
    if cfg == 3 and direction == "both":
        return "NFSGLFT nodes/sec fwd+adj at B=64"
    d = {"both": "fwd+adj", "fwd": "fwd", "adj": "adj"}[direction]
    if K > 1 and direction == "fwd":
        return f"NFSGLFT node-evaluations/sec fwd at B={B} ({K} vectors per plan)"
    return f"NFSGLFT nodes/sec {d} at B={B}"


def cpu_reference(work, rho, sample, direction="both", K=1, rank_threads=0):
    """The reference algorithm on the host (oracle port of the reference path):
    the per-call fixed stages (basal + FFT, both directions) are timed in
    full; the window loops are timed on a rho-pinned S-node sample and scaled
    to M (they are linear in the node count): T(M) = T_fixed + M * t_node."""
    from oracle import sgl_oracle as o
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    threads = o.oracle_threads() if rank_threads == 0 else rank_threads
    workers = os.cpu_count() or 1
    idx = np.linspace(0, work.M - 1, min(sample, work.M)).astype(np.int64)
    p = o.oracle_plan(work.B, work.points[idx], rho=rho)
    c = work.coeffs if work.coeffs.ndim == 1 else work.coeffs[0]
    # warm-up (thread pools, first-touch pages), excluded as the reference
    # excludes its JIT warm-up (experiments.py:240-243)
    warm = o.oracle_plan(work.B, work.points[idx[:64]], rho=rho)
    if direction in ("both", "adj"):
        o.oracle_adjoint(warm, work.values[idx[:64]], threads=threads, workers=workers)
    if direction in ("both", "fwd"):
        o.oracle_forward(warm, c, threads=threads, workers=workers)
    fw, ad = direction in ("both", "fwd"), direction in ("both", "adj")
    t_ff = t_fa = t_g = t_s = 0.0
    if fw:
        t0 = time.perf_counter()
        grid = o.spectral_forward(p, o.basal_forward(p, c), workers)
        t1 = time.perf_counter()
        o.gather(grid, p.base, p.win, p.q, threads)
        t2 = time.perf_counter()
        t_ff, t_g = t1 - t0, (t2 - t1) / len(idx)
        del grid
    if ad:
        t2 = time.perf_counter()
        g2 = o.scatter(p.grid, p.base, p.win, work.values[idx], p.q, threads)
        t3 = time.perf_counter()
        o.basal_adjoint(p, o.spectral_adjoint(p, g2, workers))
        t4 = time.perf_counter()
        t_fa, t_s = t4 - t3, (t3 - t2) / len(idx)
    nvec = K if direction == "fwd" else 1
    # one step: nvec forwards (+ one adjoint); units as the device arm counts them
    T = nvec * (t_ff + work.M * t_g) + (t_fa + work.M * t_s if ad else 0.0)
    units = work.M * nvec
    parts = []
    if fw:
        parts.append(f"forward basal+FFT {t_ff:.2f} s in full, gather {t_g * 1e6:.1f} us/node")
    if ad:
        parts.append(f"adjoint basal+FFT {t_fa:.2f} s in full, scatter {t_s * 1e6:.1f} us/node")
    return {"value": units / T, "unit": "nodes/s", "cores": int(threads), "kind": "port",
            "sample": (f"oracle port of the reference path, {direction}"
                       + (f" x {nvec} vectors" if nvec > 1 else "") + ": " + "; ".join(parts)
                       + f"; window loops timed on {len(idx)} rho-pinned nodes and scaled to M={work.M}; "
                       f"{threads} OpenMP threads, scipy.fft on {workers} workers"),
            "t_fixed_s": nvec * t_ff + t_fa, "t_node_us": (nvec * t_g + t_s) * 1e6}


STOCK = os.path.join(ROOT, "baseline", "_ref")


def stock_reference(work, rho, direction="both", K=1, s1=1000, s2=21000):
    """The unmodified reference package (baseline/_ref: numba backend, serial
    loops, pocketfft) on rho-pinned samples of s1 and s2 nodes:
    T(M) = T_fixed + M t_node per direction, plans excluded,
    JIT warm-up excluded (experiments.py:240-243).  Raises ImportError when
    the package is not installed."""
    if STOCK not in sys.path:
        sys.path.insert(0, STOCK)
    import sglnufft as ref
    c = work.coeffs if work.coeffs.ndim == 1 else work.coeffs[0]
    idx = np.linspace(0, work.M - 1, min(s2, work.M)).astype(np.int64)
    s1 = min(s1, len(idx) // 2) if len(idx) > 1 else len(idx)
    vals = work.values if work.values is not None else np.zeros(work.M, complex)
    fw, ad = direction in ("both", "fwd"), direction in ("both", "adj")
    w0 = ref.plan(work.B, work.points[idx[:16]], rho=rho)   # JIT warm-up
    if fw:
        ref.forward(w0, c)
    if ad:
        ref.adjoint(w0, vals[idx[:16]])
    t_start = time.perf_counter()
    res = {}
    for S in (s1, len(idx)):
        sel = idx[:S] if S == s1 else idx
        p = ref.plan(work.B, work.points[sel], rho=rho)
        t0 = time.perf_counter()
        if fw:
            ref.forward(p, c)
        t1 = time.perf_counter()
        if ad:
            ref.adjoint(p, vals[sel])
        t2 = time.perf_counter()
        res[S] = (t1 - t0, t2 - t1)
    S1, S2 = s1, len(idx)
    tn = [(res[S2][d] - res[S1][d]) / max(1, S2 - S1) for d in (0, 1)]
    tf = [max(0.0, res[S1][d] - S1 * tn[d]) for d in (0, 1)]
    nvec = K if direction == "fwd" else 1
    T = nvec * (tf[0] + work.M * tn[0]) * fw + (tf[1] + work.M * tn[1]) * ad
    units = work.M * nvec
    return {"value": units / T, "unit": "nodes/s", "cores": 1, "kind": "reference",
            "extrapolated": True, "sample_seconds": time.perf_counter() - t_start,
            "sample": (f"unmodified sglnufft {getattr(ref, '__version__', '')} (baseline/_ref; numba backend, serial "
                       f"loops, single-threaded pocketfft: the reference path uses one core), {direction}"
                       + (f" x {nvec} vectors" if nvec > 1 else "") +
                       f": T_fixed fwd {tf[0]:.2f} s / adj {tf[1]:.2f} s, t_node fwd {tn[0] * 1e6:.1f} us / adj "
                       f"{tn[1] * 1e6:.1f} us from rho-pinned samples of {S1} and {S2} nodes, extrapolated to "
                       f"M={work.M}; plans and JIT warm-up excluded (experiments.py:240-243)"),
            "t_fixed_s": nvec * tf[0] * fw + tf[1] * ad, "t_node_us": (nvec * tn[0] * fw + tn[1] * ad) * 1e6}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1809_10786_b200 import workloads
    w = workloads.config(args.config, M=args.points)
    direction = args.direction or {"fwd": "fwd", "adj": "adj"}.get(w.directions, "both")
    K = 1 if w.coeffs.ndim == 1 else w.coeffs.shape[0]
    steps = max(1, min(args.steps, 3))
    port = cpu_reference(w, w.rho, args.cpu_sample, direction, K)
    port_line = {k: port[k] for k in ("value", "unit", "cores", "kind", "sample")}
    vals, base, stock_err = [], None, None
    t_sample = 0.0
    try:
        if args.no_stock:
            raise ImportError("--no-stock")
        for _ in range(steps):
            r = stock_reference(w, w.rho, direction, K)
            vals.append(r["value"])
            t_sample += r["sample_seconds"]
            base = r
    except Exception as e:  # reference not importable: the oracle port stands in
        stock_err = f"{type(e).__name__}: {e}"
        vals = [port["value"]]
        base = port
    v = statistics.median(vals)
    cpu = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")}
    cpu["value"] = v
    line = {"metric": metric_name(args.config, direction, w.B, K), "impl": "reference", "value": v,
            "unit": "nodes/s",
            "n_gpus": world, "steps": len(vals), "warmup": 1,
            "ms_per_step": 1e3 * w.M * (K if direction == "fwd" else 1) / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (seeded PCG64, SURVEY 8(d))",
            "config": bench_config(w, direction, K),
            "extrapolated": True,
            "sample_seconds": t_sample if stock_err is None else None,
            "cpu_baseline": cpu, "cpu_port": port_line,
            "e2e": {"value": v, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": (("value: the unmodified reference package, timed on rho-pinned node samples and extrapolated "
                      "to M (ms_per_step is the extrapolated step, not wall time); cpu_port: the 16-thread oracle "
                      "port of the same algorithm") if stock_err is None else
                     f"reference package not importable here ({stock_err}): the oracle port stands in")}
    print(json.dumps(line), flush=True)


def bench_config(w, direction, K) -> dict:
    """The workload identity: identical in both arms (extras go to config_extra)."""
    return {"workload": w.name, "B": w.B, "M": w.M, "q": 16, "sigma": 2, "direction": direction, "vectors": K}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1809_10786_b200 as sgl
    from paper_1809_10786_b200 import _native, workloads
    from paper_1809_10786_b200.distributed import ShardedPlan, shard_indices

    # test hooks: SGL_BENCH_DEVICE pins every rank to one GPU and
    # SGL_BENCH_BACKEND=gloo replaces NCCL, so the multi-rank logic can be
    # exercised on a single-GPU box (never used for reported numbers)
    gpu = int(os.environ.get("SGL_BENCH_DEVICE", local))
    backend = os.environ.get("SGL_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    local = gpu
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    strong = args.scaling == "strong" or world == 1
    # strong: the same transform on every rank (seed 0), sharded by nodes;
    # weak: every rank its own M-node set of the config's distribution
    w = workloads.config(args.config, M=args.points, seed=0 if strong else rank)
    M_total = w.M * (1 if strong else world)
    direction = args.direction or {"fwd": "fwd", "adj": "adj"}.get(w.directions, "both")
    coeffs_h = w.coeffs                       # (count,) or (K, count) for the batched config 5
    K = 1 if coeffs_h.ndim == 1 else coeffs_h.shape[0]
    if w.values is None:
        w.values = np.zeros(w.M, dtype=complex)
    if strong and world > 1:
        # theta bands (default): whole pencil rows of the window tiles at full
        # node density on every rank (distributed.shard_indices; per-rank work
        # at N = 8: profiles/r02/shard_probe.txt)
        idx = shard_indices(w.points, rank, world, args.shard)
        w.points, w.values = w.points[idx], w.values[idx]
    pts_d = torch.as_tensor(w.points, device=dev)
    c_d = torch.as_tensor(coeffs_h, device=dev)
    v_d = torch.as_tensor(w.values, device=dev)
    # one-time process costs (loading the library and its kernel modules, the
    # cuFFT and memory-pool initialisation) are paid by a small warm-up plan,
    # as the reference's runners exclude their JIT warm-up (experiments.py:240-243)
    t0 = time.perf_counter()
    sgl.plan(w.B, pts_d[: min(w.M, 4096)], device=local, backend=args.backend).close()
    torch.cuda.synchronize()
    first_plan_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    # rho is global (all-reduce max over the ranks' shards) -- distributed.ShardedPlan
    sp = ShardedPlan(w.B, pts_d, device=local, partition=args.partition, backend=args.backend,
                     deterministic=args.deterministic) if world > 1 else None
    p = sp.plan if sp is not None else sgl.plan(w.B, pts_d, device=local, backend=args.backend,
                                                       deterministic=args.deterministic)
    rho = sp.rho if sp is not None else p.rho
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0
    pprof = sgl.plan(w.B, pts_d, rho=rho, device=local, profile=True, backend=args.backend,
                    deterministic=args.deterministic)
    stream = torch.cuda.current_stream(dev)

    def step(pl):
        f = a = None
        if direction in ("both", "fwd"):
            f = sgl.forward(pl, c_d)
        if direction in ("both", "adj"):
            if world > 1 and pl is p:   # the adjoint with its exchange step (ShardedPlan.adjoint)
                a = sp.adjoint(v_d)
            else:
                a = sgl.adjoint(pl, v_d)
        return f, a

    # per-kernel timings (CUDA events inside the library, on the launching stream)
    for _ in range(2):
        step(pprof)
    torch.cuda.synchronize()
    fw, ad = [], []
    for _ in range(3):
        step(pprof)
        torch.cuda.synchronize()
        fw.append(pprof.stage_ms("forward"))
        ad.append(pprof.stage_ms("adjoint"))
    stages_fwd = {k: statistics.median([d[k] for d in fw]) for k in fw[0]} if direction != "adj" else {}
    stages_adj = {k: statistics.median([d[k] for d in ad]) for k in ad[0]} if direction != "fwd" else {}
    stats = pprof.stats
    pprof.close()

    for _ in range(args.warmup):
        step(p)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step(p)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    units = M_total * (K if direction == "fwd" else 1)   # node evaluations of the whole job per step
    value = units / (ms / 1e3)

    # end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        c_h = torch.empty(coeffs_h.shape, dtype=torch.complex128, pin_memory=True).numpy()
        c_h[:] = coeffs_h
        v_h = torch.empty(w.values.shape, dtype=torch.complex128, pin_memory=True).numpy()
        v_h[:] = w.values
        fo = torch.empty((K * w.M,), dtype=torch.complex128, pin_memory=True).numpy()
        ao = torch.empty((p.count,), dtype=torch.complex128, pin_memory=True).numpy()
        L = _native.lib()

        def e2e_step():
            if world > 1:   # through the ShardedPlan API with host (pinned) arrays
                if direction in ("both", "fwd"):
                    _native.check(L.sgl_forward(p._handle, c_h.ctypes.data, K, fo.ctypes.data, None))
                if direction in ("both", "adj"):
                    ao[:] = sp.adjoint(v_h)
                return
            if direction == "both" and K == 1:   # one call; copies overlap the compute
                _native.check(L.sgl_forward_adjoint(p._handle, c_h.ctypes.data, fo.ctypes.data, v_h.ctypes.data,
                                                    ao.ctypes.data, None))
                return
            if direction in ("both", "fwd"):
                _native.check(L.sgl_forward(p._handle, c_h.ctypes.data, K, fo.ctypes.data, None))
            if direction in ("both", "adj"):
                _native.check(L.sgl_adjoint(p._handle, v_h.ctypes.data, ao.ctypes.data, None))

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        e_t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
        e_ms = float(e_t.item())
        fw_io, ad_io = direction in ("both", "fwd"), direction in ("both", "adj")
        e2e = {"value": units / (e_ms / 1e3), "unit": "nodes/s",
               "h2d_bytes_per_step": int(c_h.nbytes * fw_io + v_h.nbytes * ad_io),
               "d2h_bytes_per_step": int(fo.nbytes * fw_io + ao.nbytes * ad_io), "ms_per_step": e_ms}

    # roofline of the dominant kernel (algorithmic FP64 FLOPs at the FP64 peak).
    # The forward window stage runs on the int8 tensor cores when the plan
    # selected it: its algorithmic FP64-equivalent rate is reported beside the
    # executed int8 rate against the measured int8 peak.
    q = 16
    flop_per_node = 4.0 * (2 * q) ** 3     # 2 real FMAs per nonzero tap, (2q)^3 taps
    i8 = bool(stats.get("i8_gather"))
    kern = {}
    if direction in ("both", "fwd"):
        kern["gather"] = {"ms": stages_fwd["window"] / K, "flop": w.M * flop_per_node,
                          "engine": "int8 tensor cores (tcgen05.mma kind::i8, FP64 by 6x6 digit split)" if i8
                          else "FP64 DMMA (mma.sync m8n8k4)"}
    if direction in ("both", "adj"):
        i8s = bool(stats.get("i8_scatter"))
        kern["scatter"] = {"ms": stages_adj["window"], "flop": w.M * flop_per_node,
                           "engine": "int8 tensor cores (tcgen05.mma kind::i8, FP64 by 6x6 digit split)" if i8s
                           else "FP64 DMMA (mma.sync m8n8k4)"}
    for k in kern.values():
        k["tflops"] = k["flop"] / (k["ms"] * 1e-3) / 1e12
        k["frac"] = k["tflops"] / FP64_PEAK_TFLOPS
    if "gather" in kern and i8:
        g = kern["gather"]
        g["int8_tops"] = stats["i8_ksteps"] * I8_OPS_PER_KSTEP / (g["ms"] * 1e-3) / 1e12
        g["int8_frac"] = g["int8_tops"] / INT8_PEAK_TOPS
        g["int8_ops_per_launch"] = stats["i8_ksteps"] * I8_OPS_PER_KSTEP
        g["int8_useful_ops_per_launch"] = 21.0 * g["flop"]
    if "scatter" in kern and stats.get("i8_scatter"):
        g = kern["scatter"]   # same MMA shape per K-step: 21 pairs x M 128 cells x N 80 x K 32 nodes
        g["int8_tops"] = stats["i8_sksteps"] * I8_OPS_PER_KSTEP / (g["ms"] * 1e-3) / 1e12
        g["int8_frac"] = g["int8_tops"] / INT8_PEAK_TOPS
        g["int8_ops_per_launch"] = stats["i8_sksteps"] * I8_OPS_PER_KSTEP
        g["int8_useful_ops_per_launch"] = 21.0 * g["flop"]
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic = None
    try:
        if args.config == 3 and w.M == 10_000_000:   # the configuration the ncu capture was taken on
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(dom + ("_i8" if "int8_tops" in kern[dom] else ""))
    except Exception:
        pass
    if "int8_tops" in kern[dom]:
        # ALGORITHMIC ops (the verdict's definition): SURVEY 8(d)'s 4 (2q)^3 FP64 FLOP per
        # node as the 21 kept int8 digit pairs, without the tile boxes' padding; the ops
        # the kernel executes (box cells x nodes, counted from its K-steps) are beside it
        ksteps = stats["i8_ksteps"] if dom == "gather" else stats["i8_sksteps"]
        useful = kern[dom]["int8_useful_ops_per_launch"]
        ach = useful / (kern[dom]["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": INT8_PEAK_TOPS,
                "unit": "TOP/s (int8)", "frac": ach / INT8_PEAK_TOPS, "traffic": traffic,
                "peak_source": "measured tcgen05 kind::i8 peak (profiles/i8_mma_rate_r01.txt)",
                "algorithmic": f"21 digit pairs x {flop_per_node:.0f} FLOP/node x {w.M} nodes per launch",
                "executed": {"achieved": kern[dom]["int8_tops"], "frac": kern[dom]["int8_frac"],
                             "ops": f"{I8_OPS_PER_KSTEP:.0f} int8 ops per K-step x {ksteps} K-steps per launch",
                             "over_algorithmic": kern[dom]["int8_ops_per_launch"] / useful}}
    else:
        roof = {"bound": "tensor", "kernel": dom, "achieved": kern[dom]["tflops"], "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": kern[dom]["frac"], "traffic": traffic,
                "peak_source": "measured FP64 DMMA peak (profiles/fp64_peak_r01.txt); MEASURED_PEAKS.json has no FP64 figure",
                "algorithmic": f"{flop_per_node:.0f} FLOP/node x {w.M} nodes per launch"}

    # whole-step roofline: each window stage at its engine's
    # peak (FP64 FLOPs at the FP64 peak, or the int8 engines' algorithmic ops at
    # the int8 peak) + the FFTs at the HBM copy bandwidth (3 passes x
    # read+write x 16 B per cell)
    hbm_gbs = 6534.1
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_gbs = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    n_fwd, n_adj = (K if direction in ("both", "fwd") else 0), (1 if direction in ("both", "adj") else 0)
    cells = float(np.prod(p.nfft.grid_shape)) if p.nfft else 0.0
    t_gat = (21.0 * w.M * flop_per_node / (INT8_PEAK_TOPS * 1e12) if i8 else
             w.M * flop_per_node / (FP64_PEAK_TFLOPS * 1e12)) * 1e3
    t_sca = (21.0 * w.M * flop_per_node / (INT8_PEAK_TOPS * 1e12) if stats.get("i8_scatter") else
             w.M * flop_per_node / (FP64_PEAK_TFLOPS * 1e12)) * 1e3
    t_win = n_fwd * t_gat + n_adj * t_sca
    t_fft = (n_fwd + n_adj) * 3 * 2 * 16.0 * cells / (hbm_gbs * 1e9) * 1e3
    step_roof = {"t_roof_ms": t_win + t_fft, "window_ms": t_win, "fft_ms": t_fft, "frac": (t_win + t_fft) / ms,
                 "model": ("int8 window stages: algorithmic int8 ops (21 digit pairs x 4 (2q)^3 per node, no box padding) / 4550 TOP/s (tcgen05 int8 peak); " if i8 else "") +
                          "FP64 window FLOPs / 37.1 TF/s (FP64 DMMA peak) + 3-pass FFT bytes / HBM copy GB/s "
                          "(MEASURED_PEAKS.json); basal and halo work not counted"}

    cpu = cpu_port = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            r = cpu_reference(w, rho, args.cpu_sample, direction, K)
            cpu_port = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # pragma: no cover
            cpu_port = {"value": None, "unit": "nodes/s", "cores": 0, "kind": "port", "sample": f"failed: {e}"}
        cpu = cpu_port
        if not args.no_stock:
            try:   # the reference itself (baseline/_ref), when it is installed
                r = stock_reference(w, rho, direction, K)
                cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "extrapolated",
                                         "sample_seconds")}
            except Exception as e:  # pragma: no cover
                cpu_port = dict(cpu_port or {}, stock_unavailable=f"{type(e).__name__}: {e}")

    grid_gb = 16.0 * float(np.prod(p.nfft.grid_shape)) / 1e9 if p.nfft else 0.0
    node_gb = w.M * (3 * 8 * 2 + 4 * 2 + 16) / 1e9   # sorted u0..u2 + perm (gather and scatter orders) + values
    l2_note = (f"{'inputs larger than L2' if grid_gb + node_gb > 0.126 else 'working set fits L2 (126 MB)'} "
               f"(grid {grid_gb:.3g} GB, node arrays {node_gb:.3g} GB per rank)")
    if rank == 0:
        line = {
            "metric": metric_name(args.config, direction, w.B, K),
            "value": value, "unit": "nodes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded PCG64 inputs of SURVEY 8(d); no public dataset)",
            "config": bench_config(w, direction, K) | {"M": M_total},
            "config_extra": {"grid": list(p.nfft.grid_shape), "rho": rho, "l2": l2_note, "M_per_rank": w.M,
                             "deterministic_adjoint": bool(args.deterministic),
                             "parallelism": (f"{world} GPU(s), node shards ({args.shard if strong else 'own sets'}); adjoint exchange: "
                                             f"{sp.partition if sp is not None else 'none'}"
                                             + (" (coefficient all-reduce)" if sp is not None and
                                                sp.partition == "coeffs" else
                                                " (grid reduce-scatter + slab FFT)" if sp is not None else ""))},
            "e2e": e2e, "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "cpu_port": cpu_port,
            "clocks": clk,
            "gpu_launches": args.steps * ((11 if i8 else 4) * K * (direction != "adj") +
                                         (10 if stats.get("i8_scatter") else 5) * (direction != "fwd")),
            "gpu_launches_note": ("per forward vector: radial_fwd, sph_fwd, halo_fill, slab_absmax, slab_shift, "
                                  "slice_grid, tile_shift, gather_i8, absmax_c, guard_fwd, gather_tiled (gated: "
                                  "returns at once unless the guard raised its flag)" if i8 else
                                  "per forward vector: radial_fwd, sph_fwd, halo_fill, gather_tiled") +
                                 ("; per adjoint: tile_vscale, scatter_i8 (builds its value digits itself), scatter_tiled (gated), "
                                  "halo_fold, zeta_crop, sph_adj, radial_adj, sumsq_c, absmax_c, guard_adj"
                                    if stats.get("i8_scatter") else
                                    "; per adjoint: scatter_tiled, halo_fold, zeta_crop, sph_adj, radial_adj") +
                                 " (+ cuFFT and memsets, library calls)",
            "kernels": {k: {kk: vv for kk, vv in v.items() if kk != "flop"} for k, v in kern.items()},
            "stages_ms": {"forward": stages_fwd, "adjoint": stages_adj},
            "plan": {"seconds": plan_s, "warmup_plan_seconds": first_plan_s, **stats},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
