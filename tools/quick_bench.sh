#!/bin/bash
# device-only bench line (no CPU baselines) + the window-kernel stage times
python bench.py --steps 10 --warmup 3 --no-cpu --no-stock "$@" > gpurun_out/qb.json 2> gpurun_out/qb.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qb.json").read())
print("value %.4g nodes/s  ms/step %.3f  e2e %.4g" % (d["value"], d["ms_per_step"], (d.get("e2e") or {}).get("value", 0)))
for k, v in d["kernels"].items():
    print(k, "%.3f ms" % v["ms"], "int8 frac %.3f" % v.get("int8_frac", 0))
print("stages", {k: {kk: round(vv, 3) for kk, vv in v.items()} for k, v in d["stages_ms"].items()})
print("clocks", d["clocks"])
PY
