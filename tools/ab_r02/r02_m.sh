#!/bin/bash
set -u
mkdir -p gpurun_out
CMD="python tools/prof_assess.py --config large --reps 1 --sdf 2.0"
if timeout 300 $CMD > gpurun_out/m_sdf_plain.json 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:sdf -s 2 -c 2 \
      -o gpurun_out/m_sdf -f $CMD > gpurun_out/m_ncu_sdf.log 2>&1
  echo "ncu sdf rc=$?"
fi
