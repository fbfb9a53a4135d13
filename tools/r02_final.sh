#!/bin/bash
# Round-2 measurement pass: GPU tests, smoke, bench (N = 1), reference arm, GPU health after the bench,
# the ncu launch list of a short bench, then ncu --set full of one large-map and one high-res assess call (both kernels each).
# Usage: bash tools/r02_final.sh [file prefix, default H]
set -u
P=${1:-H}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${P}_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${P}_bench_reference.json 2> gpurun_out/${P}_bench_reference.err; echo "reference rc=$?"
timeout 60 nvidia-smi --query-gpu=name,clocks.sm,temperature.gpu,power.draw,memory.used --format=csv > gpurun_out/${P}_smi_after.txt 2>&1; echo "smi rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-e2e"
if timeout 600 $SMALL > gpurun_out/${P}_bench_small.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv \
      $SMALL > gpurun_out/${P}_ncu_launches.log 2>&1; echo "launch list rc=$?"
fi
CMD="python tools/prof_assess.py --config large --reps 1"
if timeout 300 $CMD > gpurun_out/${P}_large_plain.json 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 2 -c 2 \
      -o gpurun_out/${P}_large -f $CMD > gpurun_out/${P}_ncu_large.log 2>&1
  echo "ncu large rc=$?"
fi
CMD="python tools/prof_assess.py --config highres --reps 1"
if timeout 300 $CMD > gpurun_out/${P}_highres_plain.json 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 2 -c 2 \
      -o gpurun_out/${P}_highres -f $CMD > gpurun_out/${P}_ncu_highres.log 2>&1
  echo "ncu highres rc=$?"
fi
