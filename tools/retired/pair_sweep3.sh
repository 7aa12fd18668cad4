#!/bin/bash
# CTA-pair engine vs the single-CTA engine under the pair knobs (cfg3 ms/step)
run() { echo "== $*"; env "$@" timeout 300 python bench.py --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'])"; }
run BLAST_PAIR_ENGINE=0
run BLAST_PAIR_ENGINE=1
run BLAST_PAIR_ENGINE=1 BLAST_PAIR_RESCAP=0
run BLAST_PAIR_ENGINE=1 BLAST_WIDE_TILES=0
run BLAST_PAIR_ENGINE=1 BLAST_WIDE_TILES=0 BLAST_PAIR_RESCAP=0 BLAST_PAIR_STAGES=8
run BLAST_PAIR_ENGINE=1 BLAST_WIDE_TILES=0 BLAST_PAIR_STAGES=6
run BLAST_PAIR_ENGINE=1 BLAST_PAIR_R=1
