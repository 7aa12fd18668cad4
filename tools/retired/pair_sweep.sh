#!/bin/bash
# Sweep the CTA-pair engine's pipeline depth (resident weights take the rest of smem)
for st in 4 6 8 9 10 11; do
  BLAST_PAIR_STAGES=$st timeout 300 python bench.py --no-cpu --no-dense --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.load(sys.stdin); print('stages', $st, 'ms/step', round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])"
done
BLAST_DISABLE_PAIR=1 timeout 300 python bench.py --no-cpu --no-dense --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.load(sys.stdin); print('single-CTA', 'ms/step', round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])"
