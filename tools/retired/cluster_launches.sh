#!/bin/bash
# per-launch durations of the decode forward with / without the cluster-pair split (ncu, serialised)
for v in 1 0; do
  BLAST_CLUSTER_SPLIT=$v ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --clock-control none -k regex:spmm_tc --csv \
    python tools/decode_probe.py 128 0.95 2>/dev/null | grep spmm_tc | tail -6 | awk -F'","' -v v=$v '{print "CS=" v, substr($5,1,60), $(NF-2), $NF}'
done
