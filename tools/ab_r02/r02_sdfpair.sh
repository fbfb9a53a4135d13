#!/bin/bash
# SDF row pass over pairs of neighbouring cells (SE2M_SDF_PAIRS = 1) vs one cell per scan (0)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for v in sp0 sp1; do
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config large --reps 3 --sdf 2.0 | sed "s#^#$v #"
  SE2M_LIB=abx/libse2map_$v.so timeout 300 python tools/prof_assess.py --config highres --reps 3 --sdf 1.0 | sed "s#^#$v #"
done
done > gpurun_out/sdfpair_ab.txt 2>&1
SE2M_LIB=abx/libse2map_sp1.so timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py tests/test_gpu_inpaint.py -m gpu -q > gpurun_out/sdfpair_tests.log 2>&1
echo "tests rc=$?"
SE2M_LIB=abx/libse2map_sp1.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:sdf --csv \
  --log-file gpurun_out/sdfpair_launches.csv python tools/prof_assess.py --config large --reps 1 --sdf 2.0 > gpurun_out/sdfpair_ncu.log 2>&1
echo "ncu rc=$?"
