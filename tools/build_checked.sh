#!/bin/bash
# Debug build with device-side bounds checks (SE2M_CHECKS) -> abx/libse2map_checked.so (use with SE2M_LIB=...).
set -e
cd "$(dirname "$0")/.."
mkdir -p abx
C=paper_2503_02412_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DSE2M_CHECKS -Xcompiler -fPIC -shared \
     -o abx/libse2map_checked.so $C/assess.cu $C/sdf.cu $C/frontend.cu $C/inpaint.cu $C/se2map.cu -ldl
