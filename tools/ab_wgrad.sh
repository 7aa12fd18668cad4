#!/bin/bash
# wgrad item-size / schedule A/B: training step + wgrad launch times (ncu, serialised)
# usage: bash tools/ab_wgrad.sh default variants/lib_x.so ...
bash tools/ab_train.sh "$@"
for l in "$@"; do
  if [ "$l" = default ]; then unset BLAST_LIB; else export BLAST_LIB=$PWD/$l; fi
  echo "== $l wgrad launches"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wgrad --csv \
    python tools/extras_once.py train 2>/dev/null | grep wgrad | awk -F'","' '{print substr($5,1,40), $NF}' | tail -3
done
