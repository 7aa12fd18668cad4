#!/bin/bash
# per-role wait counters of the cfg3 training-step kernels (wait-counter build, diagnosis only)
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null 2>&1
BLAST_DEBUG_COUNTERS=1 python tools/extras_once.py train 2>&1 | grep "blast dbg" | tail -8
