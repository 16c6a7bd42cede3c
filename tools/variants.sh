#!/bin/bash
# A/B of experimental library builds (paper_1809_10786_b200/_lib/variants/libsgl_*.so,
# built with `python -m paper_1809_10786_b200.build --variant NAME -DX=1`):
# per variant the int8 tests (-k filter in $VTESTS), the device-only config-3
# bench line and the int8 kernels' wait counters.
mkdir -p gpurun_out/var
for lib in paper_1809_10786_b200/_lib/variants/libsgl_*.so; do
  n=$(basename $lib .so); n=${n#libsgl_}
  echo "== $n"
  export SGL_LIBRARY=$PWD/$lib
  if [ -n "$VTESTS" ]; then timeout 300 python -m pytest tests/test_i8_gpu.py -x -q $VTESTS 2>&1 | tail -2; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-stock --no-e2e > gpurun_out/var/$n.json 2> gpurun_out/var/$n.err
  python -c "
import json; d = json.loads(open('gpurun_out/var/$n.json').read())
print('value %.4g ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms'], 3) for k, v in d['kernels'].items()}, d['clocks']['sm_mhz'])
" 2>&1 | tail -1
  timeout 200 python tools/profile_run.py --m 10000000 --reps 1 --profile 2>&1 | grep -E "MMA warp|generator" | head -4
done
