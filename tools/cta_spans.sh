#!/bin/bash
# Per-CTA start/end spans of the cfg3 forward's two kernels (wait-counter build), for the
# schedule A/B: tools/cta_spans.sh  (rebuilds the library with -DBLAST_WAIT_COUNTERS first)
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null
for v in 0 1; do
  echo "== BLAST_SCHEDULE=$v"
  BLAST_SCHEDULE=$v BLAST_DEBUG_COUNTERS=1 python tools/prof_once.py 2>&1 | grep "span" | tail -2
done
python -m paper_2507_03117_b200.build --force > /dev/null
