#!/bin/bash
# wgrad sweep mode (BLAST_WG_SWEEP) A/B: training step, per-mask wgrad times, dWdown DRAM bytes
for r in 1 2 3; do for v in 1 0; do
  echo -n "WG_SWEEP=$v train: "; BLAST_WG_SWEEP=$v timeout 300 python tools/extras_quick.py train | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],4), 'ms')"
done; done
for v in 1 0; do echo "== WG_SWEEP=$v"; BLAST_WG_SWEEP=$v timeout 300 python tools/wgrad_probe.py; done
for v in 1 0; do
  echo "== WG_SWEEP=$v wgrad launches (ncu, no cache control): time, dram read"
  BLAST_WG_SWEEP=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none -k regex:wgrad_tc --csv \
    python tools/extras_once.py train 2>/dev/null | grep wgrad | awk -F'","' '{print $(NF-2), $NF}' | tail -6
done
