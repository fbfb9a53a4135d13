#!/bin/bash
# Round-2 measurement pass: GPU tests, smoke, bench (N = 1), reference arm, GPU health after the bench,
# the ncu launch list of a short bench, then ONE ncu --set full of the large-map assess call (both kernels).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/G_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/G_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/G_bench.json 2> gpurun_out/G_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/G_bench_reference.json 2> gpurun_out/G_bench_reference.err; echo "reference rc=$?"
timeout 60 nvidia-smi --query-gpu=name,clocks.sm,temperature.gpu,power.draw,memory.used --format=csv > gpurun_out/G_smi_after.txt 2>&1; echo "smi rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-e2e"
if timeout 600 $SMALL > gpurun_out/G_bench_small.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/G_launches.csv \
      $SMALL > gpurun_out/G_ncu_launches.log 2>&1; echo "launch list rc=$?"
fi
CMD="python tools/prof_assess.py --config large --reps 1"
if timeout 300 $CMD > gpurun_out/G_large_plain.json 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 2 -c 2 \
      -o gpurun_out/G_large -f $CMD > gpurun_out/G_ncu_large.log 2>&1
  echo "ncu large rc=$?"
fi
