#!/bin/bash
# bench-step overheads: strip clears in one launch; update_elevation scatter with 1 vs 4 cells per thread
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in up1 up4; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/ab_r02/stepparts.py | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
done
done > gpurun_out/steps_ab.txt 2>&1
SE2M_LIB=abx/libse2map_up4.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/steps_tests.log 2>&1
echo "tests rc=$?"
