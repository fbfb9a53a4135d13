#!/bin/bash
# GPU pass: tests on the tree library (512-thread R_T = 16 tiles), A/B vs base / c8, stream timing, ONE ncu (high-res).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g_gpu_tests.log 2>&1; echo "tests rc=$?"
for rep in 1 2; do
for v in base c8 r16; do
  lib=abx/libse2map_$v.so
  for c in highres large paper; do
    SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config $c --reps 20 | sed "s#^#$v #"
  done
  SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config highres --holes 0.02 --reps 10 | sed "s#^#$v #"
  SE2M_LIB=$lib timeout 300 python tools/prof_stream.py | sed "s#^#$v stream #"
done
done > gpurun_out/g_ab.txt 2>&1
echo "ab rc=$?"
timeout 600 python tools/prof_shards.py --configs highres > gpurun_out/g_shards.json 2> gpurun_out/g_shards.err; echo "shards rc=$?"
CMD="python tools/prof_assess.py --config highres --reps 1"
if timeout 300 $CMD > gpurun_out/g_highres_plain.json 2>&1; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 2 -c 2 \
      -o gpurun_out/g_highres -f $CMD > gpurun_out/g_ncu_highres.log 2>&1
  echo "ncu highres rc=$?"
fi
