#!/bin/bash
# per-role wait counters and per-CTA spans of the decode forward (128 tokens, 95 %), wait-counter build
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null 2>&1
BLAST_DEBUG_COUNTERS=1 python tools/decode_probe.py 128 0.95 2>&1 | grep "blast dbg" | tail -4
