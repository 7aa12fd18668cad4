#!/bin/bash
# LPT item schedule for the training gate+up (EPI_GATED_FWD_SAVE) A/B
for r in 1 2 3; do for v in 1 0; do
  echo -n "LPT_SAVE=$v train: "; BLAST_LPT_SAVE=$v timeout 300 python tools/extras_quick.py train | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],4), 'ms')"
done; done
for v in 1 0; do
  echo -n "LPT_SAVE=$v fwd-save kernel (ncu): "
  BLAST_LPT_SAVE=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spmm_tc --csv \
    python tools/extras_once.py train 2>/dev/null | grep spmm_tc | grep ", 4, " | awk -F'","' '{print $NF}' | tail -1
done
