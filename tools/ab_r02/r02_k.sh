#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/k_gpu_tests.log 2>&1; echo "tests rc=$?"
for rep in 1 2 3; do
for v in v4 v5; do
  lib=abx/libse2map_$v.so
  for c in large highres paper; do
    SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config $c --reps 20 | sed "s#^#$v #"
  done
  SE2M_LIB=$lib timeout 300 python tools/prof_stream.py | sed "s#^#$v stream #"
done
done > gpurun_out/k_ab.txt 2>&1
echo "ab rc=$?"
for c in large paper stream; do
  SE2M_LIB=abx/libse2map_phases.so timeout 300 python tools/phase_report.py --config $c
done > gpurun_out/k_phases.jsonl 2>&1
echo "phases rc=$?"
