"""bench.py's reference arm (`--impl reference`): the JSON-line contract on a
small sample, and the non-zero ranks of a torchrun launch exiting silently."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, cwd=ROOT, timeout=600)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "1", "--points", "3000",
              "--cpu-sample", "500"])
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "nodes/s"
    assert d["metric"] == "NFSGLFT nodes/sec fwd at B=16" and d["config"]["direction"] == "fwd"
    # the unmodified reference (baseline/_ref) when installed, else the oracle port
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_port"]["kind"] == "port" and d["extrapolated"] is True
    assert set(d["config"]) == {"workload", "B", "M", "q", "sigma", "direction", "vectors"}
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert abs(d["ms_per_step"] - 1e3 * 3000 / d["value"]) < 1e-6 * d["ms_per_step"]


def test_reference_arm_other_ranks_are_silent():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "1", "--points", "3000"],
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_metric_names():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.metric_name(3, "both", 64, 1) == "NFSGLFT nodes/sec fwd+adj at B=64"
    assert bench.metric_name(1, "fwd", 16, 1) == "NFSGLFT nodes/sec fwd at B=16"
    assert bench.metric_name(4, "adj", 128, 1) == "NFSGLFT nodes/sec adj at B=128"
    assert "64 vectors" in bench.metric_name(5, "fwd", 48, 64)
