#!/bin/bash
# per library variant: int8 scatter tests, the config-3 bench line, and the
# window kernels' DRAM bytes + duration from a short ncu metrics pass
mkdir -p gpurun_out/var
for lib in paper_1809_10786_b200/_lib/variants/libsgl_*.so; do
  n=$(basename $lib .so); n=${n#libsgl_}
  echo "== $n"
  export SGL_LIBRARY=$PWD/$lib
  timeout 300 python -m pytest tests/test_i8_gpu.py -x -q -k scatter 2>&1 | tail -1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-stock --no-e2e > gpurun_out/var/$n.json 2> gpurun_out/var/$n.err
  python -c "
import json; d = json.loads(open('gpurun_out/var/$n.json').read())
print('value %.4g ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms'], 3) for k, v in d['kernels'].items()}, d['clocks']['sm_mhz'])
" 2>&1 | tail -1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"k_scatter_i8" -c 1 python tools/profile_run.py --m 10000000 --reps 1 2>&1 | grep -E "dram__|gpu__time" 
done
