#!/bin/bash
# per-CTA phase timelines of the assess kernels (debug build with SE2M_PHASES) for the small configurations
set -u
mkdir -p gpurun_out
for c in paper stream large; do
  SE2M_LIB=abx/libse2map_phases.so timeout 300 python tools/phase_report.py --config $c 2>&1
done > gpurun_out/phases2.jsonl
echo done
