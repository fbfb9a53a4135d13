#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/l_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/prof_stream2.py > gpurun_out/l_stream.jsonl 2>&1; echo "stream rc=$?"
