#!/bin/bash
# per-CTA spans / role waits of the decode forward with and without the cluster-pair split
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -m paper_2507_03117_b200.build --force > /dev/null 2>&1
for v in 1 0; do
  echo "== BLAST_CLUSTER_SPLIT=$v"
  BLAST_CLUSTER_SPLIT=$v BLAST_DEBUG_COUNTERS=1 BLAST_DEBUG_CTAS=1 timeout 120 python tools/decode_probe.py 128 0.95 2>&1 | grep "blast dbg" | tail -5 | cut -c1-900
done
