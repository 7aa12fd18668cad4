#!/bin/bash
# Per-role wait counters of the cfg0 fp32 forward kernels (wait-counter build, diagnosis only)
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null 2>&1
BLAST_DEBUG_COUNTERS=1 python tools/cfg0_once.py 2>&1 | grep "blast dbg" | tail -4
