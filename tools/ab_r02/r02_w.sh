#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/w_gpu_tests.log 2>&1; echo "tests rc=$?"
for rep in 1 2; do
for v in es sr; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 20 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config large --holes 0.02 --reps 10 | sed "s#^#$v #"
done
done > gpurun_out/w_bench_ab.txt 2>&1
echo "bench ab rc=$?"
SE2M_LIB=abx/libse2map_sr.so timeout 600 python tools/prof_shards.py > gpurun_out/w_shards.json 2>&1; echo "shards rc=$?"
