#!/bin/bash
# re-tune 2: T-mode spread off, cell-entry cap 3, edge segments 8
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in base ts0 cm3 es8; do
  SE2M_LIB=abx/libse2map_$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 200 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_stream2.py 2>/dev/null | head -1 | sed "s#^#$v #"
done
done > gpurun_out/knobs2_ab.txt 2>&1
echo done
