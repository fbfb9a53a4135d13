#!/bin/bash
# launch order of the main / edge assess kernels on one-wave grids (SE2M_MAIN_FIRST): paper-like FULL, stream step
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in mf0 mf1; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 200 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_stream2.py | sed "s#^#$v #"
done
done > gpurun_out/y_ab.txt 2>&1
echo "ab rc=$?"
