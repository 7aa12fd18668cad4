#!/bin/bash
# ncu --set full of the two cfg3 MLP forward kernels (after warm-up) -> gpurun_out/ncu/
mkdir -p gpurun_out/ncu
O=gpurun_out/ncu
TAG=${1:-cur}
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:spmm_tc -s 2 -c 2 -o $O/full_$TAG -f python tools/prof_once.py > $O/ncu_$TAG.log 2>&1
tail -3 $O/ncu_$TAG.log
