#!/bin/bash
# query kernels reading / writing pinned host buffers in place (SE2M_ZERO_COPY = 1) vs staged copies (0)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in zc0 zc1; do
  SE2M_LIB=abx/libse2map_$v.so timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | sed "s#^#$v #"
done
done > gpurun_out/zc_ab.txt 2>&1
SE2M_LIB=abx/libse2map_zc1.so timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/zc_tests.log 2>&1
echo "tests rc=$?"
