#!/bin/bash
# Copy the outputs of tools/round_measure_r02.sh + tools/final_checks.sh
# (gpurun_out/r02, gpurun_out/final) into profiles/r02 and print the numbers
# the docs quote.  Run from the repo root, here (needs ncu for the summaries).
o=$PWD/gpurun_out/r02; f=$PWD/gpurun_out/final; d=$PWD/profiles/r02
python tools/ncu_quick.py $o/ncu_i8_10m.ncu-rep 25 k_scatter_i8 > $d/ncu_scatter_i8_10m_summary.txt 2>&1
python tools/ncu_quick.py $o/ncu_i8_10m.ncu-rep 25 k_gather_i8 > $d/ncu_gather_i8_10m_summary.txt 2>&1
ncu -i $o/ncu_i8_10m.ncu-rep --page raw --csv > $d/ncu_i8_10m_raw.csv 2>/dev/null
for x in bench_cfg1.json bench_cfg2.json bench_cfg3.json bench_cfg4.json bench_cfg5.json bench_ref.json gpu_tests.log launches.csv; do cp $o/$x $d/$x; done
if [ -d $f ]; then
{ echo "GPU test suite on the bounds-checked library (tools/sanitize_checked.sh: python -m paper_1809_10786_b200.build --checked; SGL_LIBRARY=.../libsgl_b200_checked.so python -m pytest tests -m gpu), final r02 build: no SGL_CHECKED trap"; tail -n 3 $f/checked_suite.log; echo; echo "compute-sanitizer on this pool: closed (profiles/r02/sanitizer_closed.txt)"; } > $d/checked_suite.txt
{ echo "tools/soak.py / tools/soak_large.py on the final r02 build (random plans, both int8 engines forced or automatic, against the generic per-node backend):"; tail -n 1 $f/soak_i8.txt; tail -n 1 $f/soak_large_i8.txt; tail -n 1 $f/soak_auto.txt; cat $d/soak_note.txt 2>/dev/null; } > $d/soak_final.txt
{ echo "torchrun --nproc-per-node 2 bench.py --gpus 2 --points 2000000 --steps 3 --warmup 3 --partition {coeffs,grid} on ONE B200 with"; echo "SGL_BENCH_DEVICE=0 SGL_BENCH_BACKEND=gloo (test hooks: both ranks on GPU 0, gloo instead of NCCL), final r02 build:"; echo "a correctness dry run of the N>1 bench path, not a scaling measurement."; for part in coeffs grid; do python -c "
import json; d = json.loads(open('$f/torchrun2_$part.json').read().strip().splitlines()[-1])
print('partition=$part: value %.4g nodes/s, n_gpus %d, %s, e2e %.4g' % (d['value'], d['n_gpus'], d['config_extra']['parallelism'], d['e2e']['value']))"; done; } > $d/torchrun2_dryrun.txt
fi
tail -n 1 $d/gpu_tests.log
python -c "
import json
for c in [1,2,3,4,5]:
    d=json.loads(open('$o/bench_cfg%d.json' % c).read())
    print(c, '%.4g'%d['value'], '%.3f ms'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], {k: round(v['ms'],3) for k,v in d['kernels'].items()}, round(d['roofline']['frac'],4), d['roofline'].get('executed',{}).get('frac'), d['clocks']['reasons'], d['gpu_launches'])
d=json.loads(open('$o/bench_ref.json').read()); print('reference arm', d['value'], d['cpu_baseline']['kind'])
"
for k in scatter gather; do echo $k; head -10 $d/ncu_${k}_i8_10m_summary.txt | grep -E "time_dur|tensor|shared_cycles|dram|fp64"; done
