#!/bin/bash
# Debug build with per-warp phase timestamps in the assess kernels (SE2M_PHASES) -> abx/libse2map_phases.so.
set -e
cd "$(dirname "$0")/.."
mkdir -p abx
C=paper_2503_02412_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DSE2M_PHASES -Xcompiler -fPIC -shared \
     -o abx/libse2map_phases.so $C/assess.cu $C/sdf.cu $C/frontend.cu $C/inpaint.cu $C/se2map.cu -ldl
