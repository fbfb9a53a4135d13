#!/bin/bash
# GPU pass: tests, A/B (abx/libse2map_base.so = previous build) of the assess timings, shards, ONE ncu (high-res).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/e_gpu_tests.log 2>&1; echo "tests rc=$?"
for rep in 1 2; do
for lib in abx/libse2map_base.so paper_2503_02412_b200/libse2map.so; do
  for c in highres large; do
    SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config $c --reps 20 | sed "s#^#$lib #"
  done
  SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config highres --holes 0.02 --reps 10 | sed "s#^#$lib #"
  SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config highres --segments 1 --reps 20 | sed "s#^#$lib #"
done
done > gpurun_out/e_ab.txt 2>&1
echo "ab rc=$?"
timeout 600 python tools/prof_shards.py --configs highres > gpurun_out/e_shards.json 2> gpurun_out/e_shards.err; echo "shards rc=$?"
CMD="python tools/prof_assess.py --config highres --reps 1"
if timeout 300 $CMD > gpurun_out/e_highres_plain.json 2>&1; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 1 -c 1 \
      -o gpurun_out/e_highres -f $CMD > gpurun_out/e_ncu_highres.log 2>&1
  echo "ncu highres rc=$?"
fi
