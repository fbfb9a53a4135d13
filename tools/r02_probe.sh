#!/bin/bash
# Round-2 first GPU pass: GPU tests, the compute-sanitizer tier, ncu of the high-res assess kernel and
# of the paper-like / stream configurations.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/p_smi_before.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/p_gpu_tests.log 2>&1; echo "tests rc=$?"
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py all \
      > gpurun_out/p_san_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"
done
timeout 600 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_cases.py tiny chain step \
    > gpurun_out/p_san_initcheck.log 2>&1; echo "sanitizer initcheck rc=$?"
if timeout 300 python tools/prof_assess.py --config highres --reps 5 > gpurun_out/p_highres.json 2>&1; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 2 -c 1 \
      -o gpurun_out/p_highres -f python tools/prof_assess.py --config highres --reps 1 > gpurun_out/p_ncu_highres.log 2>&1
  echo "ncu highres rc=$?"
fi
if timeout 300 python tools/prof_assess.py --config paper --reps 20 > gpurun_out/p_paper.json 2>&1; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:assess_kernel -s 3 -c 1 \
      -o gpurun_out/p_paper -f python tools/prof_assess.py --config paper --reps 1 > gpurun_out/p_ncu_paper.log 2>&1
  echo "ncu paper rc=$?"
fi
if timeout 300 python tools/prof_stream.py > gpurun_out/p_stream.txt 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
      --log-file gpurun_out/p_stream_launches.csv python tools/prof_stream.py > gpurun_out/p_ncu_stream.log 2>&1
  echo "ncu stream rc=$?"
fi
nvidia-smi --query-gpu=name,clocks.sm,temperature.gpu,power.draw --format=csv > gpurun_out/p_smi_after.txt 2>&1
echo "smi rc=$?"
