#!/bin/bash
# GPU pass: A/B v2 (R16, 64-bit seg math in the kernel) vs v3 (tree: segment tables); phase timelines (debug build).
set -u
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in v2 v3; do
  lib=abx/libse2map_$v.so
  for c in large highres paper; do
    SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config $c --reps 20 | sed "s#^#$v #"
  done
  SE2M_LIB=$lib timeout 300 python tools/prof_stream.py | sed "s#^#$v stream #"
done
done > gpurun_out/i_ab.txt 2>&1
echo "ab rc=$?"
for c in paper stream large; do
  SE2M_LIB=abx/libse2map_phases.so timeout 300 python tools/phase_report.py --config $c
done > gpurun_out/i_phases.jsonl 2>&1
echo "phases rc=$?"
