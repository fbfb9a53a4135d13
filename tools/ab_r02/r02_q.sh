#!/bin/bash
set -u
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in r01 m0s0 m0s0b; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
done
done > gpurun_out/q_bench_ab.txt 2>&1
echo "bench ab rc=$?"
