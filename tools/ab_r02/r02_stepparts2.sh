#!/bin/bash
# bench-step overheads after: strip clears as one 1-D launch over both strips, 4-cell scatter, no counter reset in the
# zero-copy async queries
set -u
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 300 python tools/ab_r02/stepparts.py | sed "s#^#cur #"
  timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#cur #"
  timeout 300 python tools/prof_stream2.py 2>/dev/null | head -1 | sed "s#^#cur #"
done > gpurun_out/steps2_ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/steps2_tests.log 2>&1
echo "tests rc=$?"
