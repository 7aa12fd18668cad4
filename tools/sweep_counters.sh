#!/bin/bash
# per-role wait counters for one cfg3-shape point (block $1, sparsity $2), wait-counter build
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null 2>&1
BLAST_DEBUG_COUNTERS=1 python tools/sweep_point.py $1 $2 2 2>&1 | grep "blast dbg" | tail -4
