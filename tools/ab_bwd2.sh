#!/bin/bash
# 256-token gating backward (BLAST_WIDE_BWD2) A/B: cfg3 training step + per-kernel launch times
for r in 1 2 3; do for v in 1 0; do
  echo -n "WIDE_BWD2=$v train: "; BLAST_WIDE_BWD2=$v timeout 300 python tools/extras_quick.py train | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],4), 'ms')"
done; done
for v in 1 0; do
  echo "== WIDE_BWD2=$v launch list (ncu, serialised)"
  BLAST_WIDE_BWD2=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spmm_tc --csv \
    python tools/extras_once.py train 2>/dev/null | grep spmm_tc | awk -F'","' '{print substr($5,1,90), $NF}' | tail -6
done
