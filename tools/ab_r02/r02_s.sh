#!/bin/bash
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in r01 d2 tm; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
done
done > gpurun_out/s_bench_ab.txt 2>&1
echo "bench ab rc=$?"
for v in d2 tm; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python tools/prof_shards.py --configs large | sed "s#^#$v #"
done > gpurun_out/s_shards.txt 2>&1
echo "shards rc=$?"
for v in r01 d2 tm; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config large --reps 2 > /dev/null 2>&1 && \
  SE2M_LIB=abx/libse2map_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:assess_kernel --csv \
     --log-file gpurun_out/s_launch_$v.csv python tools/prof_assess.py --config large --reps 2 > /dev/null 2>&1
  echo "ncu $v rc=$?"
done
