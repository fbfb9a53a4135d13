#!/bin/bash
# high-res: the edge kernel's own chain segments (12 / 18 vs the main chain's 8)
set -u
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in base es12 es18; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
done
done > gpurun_out/hres_edge.txt 2>&1
echo done
