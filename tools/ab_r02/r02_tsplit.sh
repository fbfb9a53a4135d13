#!/bin/bash
# vertical-window-edge tiles in their own kernel (SE2M_TSPLIT = 1) vs in the main kernel (0), per configuration
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in ts1 ts0; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 20 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config large --reps 10 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 200 | sed "s#^#$v #"
done
done > gpurun_out/tsplit_ab.txt 2>&1
echo done
