#!/bin/bash
# programmatic dependent launch (map-update kernels trigger, the assess kernel waits before reading heights) vs off
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in pdl0 pdl1; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_stream2.py | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 200 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
done
done > gpurun_out/pdl_ab.txt 2>&1
SE2M_LIB=abx/libse2map_pdl1.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pdl_tests.log 2>&1
echo "tests rc=$?"
