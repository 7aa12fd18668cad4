#!/bin/bash
# ncu --set full of the decode-size (128 tokens, 95 %) gate+up and down kernels -> gpurun_out/ncu/
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_tc -s 6 -c 2 -o gpurun_out/ncu/decode_${1:-cur} -f python tools/decode_probe.py 128 0.95 > gpurun_out/ncu/decode.log 2>&1
tail -2 gpurun_out/ncu/decode.log
