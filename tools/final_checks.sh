#!/bin/bash
# Final-build evidence: the GPU suite on the bounds-checked library, the soak of
# random plans with both int8 engines forced, and the N = 2 bench dry run under
# torchrun (test hooks: both ranks on GPU 0, gloo) for both adjoint partitions.
o=gpurun_out/final
mkdir -p $o
bash tools/sanitize_checked.sh $o > $o/checked_tail.txt 2>&1
PYTHONPATH=$PWD python tools/soak.py 800 i8 > $o/soak_i8.txt 2>&1
PYTHONPATH=$PWD python tools/soak_large.py 60 i8 > $o/soak_large_i8.txt 2>&1
for part in coeffs grid; do
  SGL_BENCH_DEVICE=0 SGL_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --points 2000000 --steps 3 --warmup 3 --no-cpu \
    --partition $part > $o/torchrun2_$part.json 2> $o/torchrun2_$part.err
done
tail -3 $o/checked_suite.log; tail -1 $o/soak_i8.txt; tail -1 $o/soak_large_i8.txt
for part in coeffs grid; do python -c "
import json; d = json.loads(open('$o/torchrun2_$part.json').read().strip().splitlines()[-1])
print('$part', '%.4g' % d['value'], d['n_gpus'], d['config_extra']['parallelism'], 'e2e %.4g' % d['e2e']['value'])"; done
