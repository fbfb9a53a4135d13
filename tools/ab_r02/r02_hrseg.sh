#!/bin/bash
# high-res yaw-chain segments S = 1 / 2 / 4 / 8 / 12: one-GPU time and the yaw-shard balance at G = 2, 4, 8
set -u
mkdir -p gpurun_out
for S in 1 2 4 8 12; do
  timeout 300 python tools/prof_assess.py --config highres --reps 20 --segments $S | sed "s#^#S$S #"
  timeout 600 python tools/prof_shards.py --configs highres --segments $S | sed "s#^#S$S #"
done > gpurun_out/hrseg.txt 2>&1
echo done
