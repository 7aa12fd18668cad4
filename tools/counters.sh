#!/bin/bash
# Per-role wait counters of the tensor-core engines on the GPU box:
# build with -DBLAST_WAIT_COUNTERS locally, run tools/dbg_run.py there, rebuild normally.
set -e
cd "$(dirname "$0")/.."
rm -rf paper_2507_03117_b200/_build
BLAST_NVCC_FLAGS=-DBLAST_WAIT_COUNTERS python -c "from paper_2507_03117_b200 import build; build.build(force=True)" > /dev/null
/usr/local/graft/bin/gpurun --timeout 600 -- 'BLAST_DEBUG_COUNTERS=1 python tools/dbg_run.py > gpurun_out/dbg.txt 2>&1' | tail -1
rm -rf paper_2507_03117_b200/_build
python -c "from paper_2507_03117_b200 import build; build.build(force=True)" > /dev/null
grep "blast dbg" gpurun_out/dbg.txt | head -2
