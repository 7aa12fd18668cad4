#!/bin/bash
# Decode-regime diagnosis (cfg3 shape at 95 %, m tokens): per-CTA spans of the two kernels
# (wait-counter build), then graph replay times with the normal build.
m=${1:-128}
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null
BLAST_DEBUG_COUNTERS=1 python tools/decode_probe.py $m 0.95 2>&1 | grep "blast dbg" | tail -4
python -m paper_2507_03117_b200.build --force > /dev/null
python tools/graph_probe.py
