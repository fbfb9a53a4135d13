#!/bin/bash
# GPU pass: large-map A/B (base / v1 = tree / v2 = tree + 64-bit seg math), then the bench on the tree library.
set -u
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in base v1 v2; do
  lib=abx/libse2map_$v.so
  SE2M_LIB=$lib timeout 300 python tools/prof_assess.py --config large --reps 20 | sed "s#^#$v #"
done
done > gpurun_out/h_ab.txt 2>&1
echo "ab rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench rc=$?"
timeout 60 nvidia-smi --query-gpu=name,clocks.sm,temperature.gpu,power.draw,memory.used --format=csv > gpurun_out/h_smi.txt 2>&1; echo "smi rc=$?"
