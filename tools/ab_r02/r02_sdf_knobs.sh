#!/bin/bash
# SDF pass geometry: row-pass cells per thread (SE2M_SDF_CPT 2 / 4 / 8), column-pass segment rows (SE2M_SDF_SEG 64 / 128)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in s0 c2 c8 g64; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config large --reps 3 --sdf 2.0 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 3 --sdf 1.0 | sed "s#^#$v #"
done
done > gpurun_out/sdfk_ab.txt 2>&1
echo done
