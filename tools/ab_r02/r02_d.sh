#!/bin/bash
# GPU pass: tests on the new library, A/B (abx/libse2map_base.so = previous commit) of the assess timings.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/d_gpu_tests.log 2>&1; echo "tests rc=$?"
for rep in 1 2; do
for lib in abx/libse2map_base.so paper_2503_02412_b200/libse2map.so; do
  for c in large highres paper; do
    SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config $c --reps 20 | sed "s#^#$lib #"
  done
  SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config large --holes 0.02 --reps 10 | sed "s#^#$lib #"
done
done > gpurun_out/d_ab.txt 2>&1
echo "ab rc=$?"
timeout 600 python tools/prof_shards.py --configs large > gpurun_out/d_shards.json 2> gpurun_out/d_shards.err; echo "shards rc=$?"
