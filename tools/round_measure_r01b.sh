# round-1 measurement after the int8 gather: bench lines, launch list, ncu full captures
set -x
python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
for c in 1 2 4 5; do python bench.py --config $c > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/profile_run.py --m 10000000 --reps 1 > gpurun_out/pr.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_gather_i8|k_scatter_i8" -c 2 -o gpurun_out/ncu_window_10m python tools/profile_run.py --m 10000000 --reps 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
