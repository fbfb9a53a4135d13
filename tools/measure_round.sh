#!/bin/bash
# One measurement pass on a GPU box (run through gpurun from the repo root); outputs in gpurun_out/:
#   gpu_tests.log, smoke.log, bench.json (+ .err), bench_reference.json, launches.csv (ncu launch list of the same
#   bench command, cold-cache / serialised), smi_after.txt (the GPU still answers after the bench).
# At most one ncu pass per gpurun call (B200_PROFILING.md); each only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?; echo "bench rc=$rc"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference rc=$?"
timeout 60 nvidia-smi --query-gpu=name,clocks.sm,temperature.gpu,power.draw,memory.used --format=csv > gpurun_out/smi_after.txt 2>&1
echo "smi after bench rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-e2e"
if timeout 600 $SMALL > gpurun_out/bench_small.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
      $SMALL > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
fi
