#!/bin/bash
# A/B of the current library against _lib/variants/libsgl_base.so: int8 /
# determinism / guard tests on the current build, then the device-only
# config-3 bench line and the scatter wait counters for both.
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_i8_gpu.py tests/test_determinism_gpu.py tests/test_guard_gpu.py tests/test_parity_scale_gpu.py -x -q 2>&1 | tail -3
for n in cur base; do
  if [ $n = base ]; then export SGL_LIBRARY=$PWD/paper_1809_10786_b200/_lib/variants/libsgl_base.so; fi
  [ $n = base ] && [ ! -f "$SGL_LIBRARY" ] && continue
  echo "== $n"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-stock --no-e2e > gpurun_out/ab/$n.json 2> gpurun_out/ab/$n.err
  python -c "
import json; d = json.loads(open('gpurun_out/ab/$n.json').read())
print('value %.4g ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms'], 3) for k, v in d['kernels'].items()}, d['clocks']['sm_mhz'])
" 2>&1 | tail -1
  timeout 200 python tools/profile_run.py --m 10000000 --reps 1 --profile 2>&1 | grep -E "scatter (MMA warp|generator)" | head -4
done
