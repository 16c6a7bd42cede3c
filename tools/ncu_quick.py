"""Quick text summary of an ncu --set full report: duration, pipe utilisation, stalls, hottest SASS lines."""
import csv, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + kf, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[-1]
m = {k: (vv, uu) for k, uu, vv in zip(h, u, v)}
keys = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in m: print(f"{k:80s} {m[k][0]} {m[k][1]}")
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio"):
        try:
            if float(m[k][0]) > 0.1: print(f"  stall {k[34:-23]:30s} {m[k][0]}")
        except ValueError: pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kf, capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows[:5]) if "Source" in r][0]
hdr = rows[hi]; isrc = hdr.index("Source"); ia = hdr.index("Address"); ws = hdr.index("Warp Stall Sampling (All Samples)")
# per-PC stall reasons (sampled), the top three of each hot line
reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try: return float(x.replace(",", ""))
    except ValueError: return 0.0


data = []
for r in rows[hi + 1:]:
    try: data.append((float(r[ws].replace(",", "")), r[ia][-5:], r[isrc][:70], r))
    except ValueError: pass
tot = sum(d[0] for d in data) or 1
for s, a, t, r in sorted(data, key=lambda d: -d[0])[:top]:
    rs = sorted(((num(r[i]), n) for i, n in reasons), reverse=True)[:3]
    why = " ".join(f"{n}={100 * v / s:.0f}%" for v, n in rs if v > 0) if s else ""
    print(f"{100*s/tot:5.1f}% {a} {t:70s} {why}")
