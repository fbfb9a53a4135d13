#!/bin/bash
# One measurement pass on a GPU box (run through gpurun from the repo root); outputs in gpurun_out/:
#   gpu_tests.log, bench.json (+ .err), bench_reference.json, launches.csv (ncu launch list of the same
#   bench command, cold-cache / serialised), bench_assess.ncu-rep (ncu --set full of the two kernels of one assess call).
# Each ncu pass runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?; echo "bench rc=$rc"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-e2e"
if $SMALL > gpurun_out/bench_small.json 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
      $SMALL > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
  ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 6 -c 2 \
      -o gpurun_out/bench_assess -f $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
