#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the window kernels on small goldens
# (tools/min_case.py): int8 gather + scatter (+ guard and gated FP64 kernels), FP64 tiled kernels.
out=${1:-gpurun_out}
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/min_case.py b8_q16 i8 > $out/plain.log 2>&1 || { echo "plain run failed"; cat $out/plain.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  for case in "b8_q16 i8" "b8_q16 tiled" "b12_q12 i8" "edges_b4_q5 i8"; do
    echo "=== $tool: $case" >> $out/sanitizer_$tool.log
    timeout 900 $CS --tool $tool --print-limit 20 python tools/min_case.py $case >> $out/sanitizer_$tool.log 2>&1
    echo "exit $?" >> $out/sanitizer_$tool.log
  done
done
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|=== |exit" $out/sanitizer_*.log
