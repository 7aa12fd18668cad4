#!/bin/bash
# A/B of the decode forward (graph replay, L2 flushed and warm) with and without the hand-off
for r in 1 2 3; do for v in 1 0; do echo -n "HAND_OFF=$v "; BLAST_HAND_OFF=$v python tools/extras_quick.py decode | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['us'],2), 'us flushed')"; done; done
for v in 1 0; do echo -n "HAND_OFF=$v warm: "; BLAST_HAND_OFF=$v python tools/graph_probe.py 2>&1 | head -1; done
