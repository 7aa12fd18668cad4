#!/bin/bash
# per-role wait counters for one cfg3-shape point (block $1, sparsity $2), both BLAST_MULTI_BLOCK settings
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null 2>&1
for mb in 0 1; do echo "BLAST_MULTI_BLOCK=$mb"; BLAST_MULTI_BLOCK=$mb BLAST_DEBUG_COUNTERS=1 python tools/sweep_point.py $1 $2 2 2>&1 | grep "blast dbg" | tail -4; done
