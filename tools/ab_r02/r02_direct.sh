#!/bin/bash
# how much of the small-map latency is the FP64 direct path (footprints with < 32 known cells)? (diagnostic:
# SE2M_DIRECT_N = 0 disables it, parity not expected)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in pdl1 d2; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_stream2.py 2>/dev/null | head -1 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config paper --reps 200 | sed "s#^#$v #"
done
done > gpurun_out/direct_ab.txt 2>&1
echo done
SE2M_LIB=abx/libse2map_d2.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/d2_tests.log 2>&1
echo "tests rc=$?"
