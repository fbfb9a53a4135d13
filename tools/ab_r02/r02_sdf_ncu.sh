#!/bin/bash
# ncu --set full of the two SDF kernels (NEXT-2) on the large map after the round-2 rework
set -u
mkdir -p gpurun_out
CMD="python tools/prof_assess.py --config large --reps 1 --sdf 2.0"
if timeout 300 $CMD > gpurun_out/sdfn_plain.json 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:sdf -c 2 \
      -o gpurun_out/sdfn -f $CMD > gpurun_out/sdfn_ncu.log 2>&1
  echo "ncu rc=$?"
fi
