#!/bin/bash
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in r01 cur m0 m0s0; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config large --holes 0.02 --reps 10 | sed "s#^#$v #"
done
done > gpurun_out/p_bench_ab.txt 2>&1
echo "bench ab rc=$?"
