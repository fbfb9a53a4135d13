#!/bin/bash
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in r01 v6 sdfnew; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
done
done > gpurun_out/n_bench_ab.txt 2>&1
echo "bench ab rc=$?"
for rep in 1 2; do
for v in sdfold sdfnew; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config large --reps 5 --sdf 2.0 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 5 --sdf 1.0 | sed "s#^#$v #"
done
done > gpurun_out/n_sdf_ab.txt 2>&1
echo "sdf ab rc=$?"
timeout 600 python -m pytest tests/test_gpu_next.py -q -x > gpurun_out/n_next_tests.log 2>&1; echo "next tests rc=$?"
