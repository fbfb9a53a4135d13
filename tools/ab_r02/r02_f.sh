#!/bin/bash
# GPU pass: bounds-checked library over the sanitizer cases + GPU tests; unroll A/B; ONE ncu (stream step).
set -u
mkdir -p gpurun_out
SE2M_LIB=abx/libse2map_checked.so timeout 900 python tools/sanitize_cases.py all > gpurun_out/f_checked_cases.log 2>&1; echo "checked cases rc=$?"
SE2M_LIB=abx/libse2map_checked.so timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f_checked_tests.log 2>&1; echo "checked tests rc=$?"
for rep in 1 2; do
for v in base c4 c8 p4c4 p1c4; do
  lib=abx/libse2map_$v.so
  for c in large highres; do
    SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config $c --reps 20 | sed "s#^#$v #"
  done
  SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config large --holes 0.02 --reps 10 | sed "s#^#$v #"
done
done > gpurun_out/f_ab.txt 2>&1
echo "ab rc=$?"
if timeout 300 python tools/prof_stream.py > gpurun_out/f_stream_plain.txt 2>&1; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 200 -c 2 \
      -o gpurun_out/f_stream -f python tools/prof_stream.py > gpurun_out/f_ncu_stream.log 2>&1
  echo "ncu stream rc=$?"
fi
