#!/bin/bash
# LPT item schedule for the inference gate+up (BLAST_LPT_GU) A/B on the cfg3 bench
# (the BLAST_LPT_GU switch was removed after this A/B: neutral on cfg3)
for r in 1 2 3; do for v in 1 0; do
  echo -n "LPT_GU=$v: "; BLAST_LPT_GU=$v python bench.py --steps 30 --warmup 5 --no-extras --no-cpu --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'ms', {k: round(v,4) for k,v in d['mlp_roofline']['kernel_ms'].items()})"
done; done
