#!/bin/bash
run() { env "$@" timeout 300 python bench.py --no-cpu --no-dense --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.load(sys.stdin); print('$*', d['mlp_roofline']['kernel_ms'])"; }
run BLAST_PAIR_STAGES=8 BLAST_PAIR_RESCAP=0
run BLAST_PAIR_STAGES=8 BLAST_PAIR_R=32
run BLAST_PAIR_STAGES=8 BLAST_PAIR_R=1
run BLAST_PAIR_STAGES=8 BLAST_PAIR_R=2
run BLAST_PAIR_STAGES=6 BLAST_PAIR_R=4
run BLAST_PAIR_STAGES=8 BLAST_PAIR_R=1 BLAST_PAIR_RESCAP=0
