#!/bin/bash
# Round-2 measurement: GPU suite, bench lines for every config, the reference
# arm, the ncu launch list of the default bench command, and ncu --set full
# captures of both int8 window kernels at config 3 (1e7 nodes).
o=gpurun_out/r02
mkdir -p $o
python -m pytest tests -m gpu -q 2>&1 | tail -5 > $o/gpu_tests.log
python bench.py > $o/bench_cfg3.json 2> $o/bench_cfg3.err
for c in 1 2 4 5; do python bench.py --config $c --no-stock > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err; done
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-stock --no-e2e > $o/ncu_launch.log 2>&1
python tools/profile_run.py --m 10000000 --reps 1 > $o/pr.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_gather_i8|k_scatter_i8" -c 2 \
    -o $o/ncu_i8_10m python tools/profile_run.py --m 10000000 --reps 1 > $o/ncu_full.log 2>&1
tail -2 $o/ncu_full.log
