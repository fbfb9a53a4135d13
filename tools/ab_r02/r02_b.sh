#!/bin/bash
# GPU pass: tests, per-rank shard timing, bench, then ONE ncu (the high-res assess kernel).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/b_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/prof_shards.py > gpurun_out/b_shards.json 2> gpurun_out/b_shards.err; echo "shards rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "bench rc=$?"
nvidia-smi --query-gpu=name,clocks.sm,temperature.gpu,power.draw --format=csv > gpurun_out/b_smi.txt 2>&1; echo "smi rc=$?"
CMD="python tools/prof_assess.py --config highres --reps 1"
if timeout 300 $CMD > gpurun_out/b_highres_plain.json 2>&1; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 1 -c 1 \
      -o gpurun_out/b_highres -f $CMD > gpurun_out/b_ncu_highres.log 2>&1
  echo "ncu highres rc=$?"
fi
