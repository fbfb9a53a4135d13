#!/bin/bash
# GPU pass: tests, chain-segment A/B on high-res and large, per-rank shard timing, ONE ncu (large assess).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/c_gpu_tests.log 2>&1; echo "tests rc=$?"
for s in 1 2 4 8 36; do timeout 300 python tools/prof_assess.py --config highres --reps 20 --segments $s; done > gpurun_out/c_seg_highres.jsonl 2>&1
for s in 1 2 4 8; do timeout 300 python tools/prof_assess.py --config large --reps 10 --segments $s; done > gpurun_out/c_seg_large.jsonl 2>&1
echo "segments rc=$?"
timeout 600 python tools/prof_shards.py > gpurun_out/c_shards.json 2> gpurun_out/c_shards.err; echo "shards rc=$?"
CMD="python tools/prof_assess.py --config large --reps 1"
if timeout 300 $CMD > gpurun_out/c_large_plain.json 2>&1; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 2 -c 2 \
      -o gpurun_out/c_large -f $CMD > gpurun_out/c_ncu_large.log 2>&1
  echo "ncu large rc=$?"
fi
