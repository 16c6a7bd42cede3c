"""Summarise `ncu --set full` exports of the window kernels for profiles/.

    python tools/ncu_summary.py gather profiles/r01/ncu_gather_10m_raw.csv /tmp/src_gather.csv
    python tools/ncu_summary.py scatter profiles/r01/ncu_scatter_10m_raw.csv /tmp/src_scatter.csv

Writes profiles/r01/ncu_<kernel>_10m_summary.txt and updates
profiles/ncu_traffic.json (DRAM bytes per launch -> bench.py roofline.traffic).
The raw CSV is `ncu -i X --page raw --csv`, the source CSV
`ncu -i X --page source --csv --print-source sass`.
"""
import csv
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SMSPS = 148 * 4
ALGO_DMMA = 1e7 * 32 * 8   # 1e7 nodes x 32 slabs x (32 x 32 x 2 / 256) DMMAs per node-slab


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, units, val = rows[0], rows[1], rows[-1]
    m = {h: (num(v), u) for h, u, v in zip(hdr, units, val)}

    def get(k, scale_to=None):
        v, u = m.get(k, (0.0, ""))
        if scale_to == "GB":
            v *= {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1.0)
        if scale_to == "ms":
            v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1.0)
        return v
    return get


def stall_table(path, top=8):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    ci = [hdr.index(c) for c in cols]
    isrc = hdr.index("Source")
    seen, data = set(), []
    for r in rows[2:]:
        if len(r) <= max(ci) or r[0] in seen:
            continue
        seen.add(r[0])
        data.append(r)
    tot = {c: sum(num(r[i]) for r in data) for c, i in zip(cols, ci)}
    T = sum(tot.values()) or 1.0
    reasons = sorted(((v / T * 100, c[6:]) for c, v in tot.items()), reverse=True)
    allc = hdr.index("Warp Stall Sampling (All Samples)")
    hot = sorted(data, key=lambda r: -num(r[allc]))[:top]
    S = sum(num(r[allc]) for r in data) or 1.0
    return reasons, [(num(r[allc]) / S * 100, r[isrc].strip()) for r in hot]


def main():
    kern, raw, src = sys.argv[1], sys.argv[2], sys.argv[3]
    g = raw_metrics(raw)
    ms = g("gpu__time_duration.sum", "ms")
    rd, wr = g("dram__bytes_read.sum", "GB"), g("dram__bytes_write.sum", "GB")
    tensor = g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    fp64 = g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
    dmma = g("SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg") * SMSPS / 16.0
    inst = g("smsp__inst_executed.sum")
    reasons, hot = stall_table(src)
    lines = [f"{kern}: ncu --set full, M = 1e7 (config-3 shape), one launch",
             f"  duration                  {ms:.3f} ms",
             f"  tensor (DMMA) pipe active {tensor:.1f} %   fp64 (DFMA/DMUL) pipe {fp64:.1f} %",
             f"  DMMAs executed            {dmma:.3e}  = {dmma / ALGO_DMMA:.3f} x algorithmic",
             f"  warp instructions         {inst:.3e}",
             f"  DRAM read / write         {rd:.3f} / {wr:.3f} GB",
             f"  registers / thread        {g('launch__registers_per_thread'):.0f}",
             "  stall reasons: " + ", ".join(f"{c} {v:.1f}%" for v, c in reasons[:7]),
             "  hottest SASS (share of stall samples):"]
    lines += [f"    {v:5.1f}%  {s[:70]}" for v, s in hot]
    out = os.path.join(ROOT, "profiles", "r01", f"ncu_{kern}_10m_summary.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {"detail": {}}
    d[kern] = (rd + wr) * 1e9
    d.setdefault("detail", {})[kern] = {
        "duration_ms": ms, "dram_read_GB": rd, "dram_write_GB": wr, "dmma_pipe_active": tensor / 100,
        "dmma_count": dmma, "inst": inst, "traffic_GB": rd + wr, "structural_factor": dmma / ALGO_DMMA,
        "source": f"profiles/r01/ncu_{kern}_10m_* (ncu --set full, M=1e7, config-3 shape)"}
    json.dump(d, open(tj, "w"), indent=1)


if __name__ == "__main__":
    main()
