#!/bin/bash
# window-kernel times per BASELINE config and engine choice (device bench, no CPU legs)
for c in 1 2 3 4 5; do
  for b in auto tiled i8; do
    python bench.py --config $c --backend $b --steps 5 --warmup 3 --no-cpu --no-stock --no-e2e > gpurun_out/es.json 2>/dev/null
    python -c "
import json; d = json.loads(open('gpurun_out/es.json').read())
print('cfg$c', '$b', 'ms/step %.3f' % d['ms_per_step'], {k: round(v['ms'], 3) for k, v in d['kernels'].items()}, 'i8s', d['plan']['i8_scatter'])
"
  done
done
