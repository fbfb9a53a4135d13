#!/bin/bash
# high-res: the edge kernel with fewer chain segments than the main chain (4 / 2 / 1 vs 8)
set -u
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in el8 el4 el2 el1; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
done
done > gpurun_out/hres_edge2.txt 2>&1
echo done
for v in el8 el4; do SE2M_LIB=abx/libse2map_$v.so timeout 600 python tools/prof_shards.py --configs highres | sed "s#^#$v #"; done >> gpurun_out/hres_edge2.txt 2>&1
