#!/bin/bash
# multi-wave edge grids: edge kernel on the map stream with programmatic launch, main kernel on the forked stream (SE2M_EDGE_ON_MAIN = 1) vs the reverse (0)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in em0 em1; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 200 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_stream2.py 2>/dev/null | sed "s#^#$v #"
done
done > gpurun_out/em_ab.txt 2>&1
SE2M_LIB=abx/libse2map_em1.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/em_tests.log 2>&1
echo "tests rc=$?"
