#!/bin/bash
# re-tune after the border unroll: interior prefix unroll 4, R_T = 8 cell unroll 4, edge segments 2, direct-loop unroll 4
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in base up4 uc4 es2 dl4; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 200 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_stream2.py 2>/dev/null | head -1 | sed "s#^#$v #"
done
done > gpurun_out/knobs_ab.txt 2>&1
echo done
