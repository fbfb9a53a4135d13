#!/bin/bash
# pair-row h^ plane in the row-mode kernel (one 8-byte load per cell entry for both states of a pair) vs the current build
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in mf1 hp; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
done
done > gpurun_out/z_ab.txt 2>&1
SE2M_LIB=abx/libse2map_hp.so timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/z_tests.log 2>&1
echo "tests rc=$?"
