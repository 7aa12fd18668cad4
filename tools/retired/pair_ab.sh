# CTA-pair engine (single output staging buffer, 5 panel stages) vs the single-CTA engine
run() { echo "== $*"; env "$@" timeout 300 python bench.py --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])"; }
timeout 900 python -m pytest tests/test_gpu_modes.py -q -x 2>&1 | tail -1
run BLAST_PAIR_ENGINE=0
run BLAST_PAIR_ENGINE=1 BLAST_PAIR_RESCAP=0 BLAST_PAIR_STAGES=5
run BLAST_PAIR_ENGINE=1 BLAST_PAIR_STAGES=5
run BLAST_PAIR_ENGINE=0
run BLAST_PAIR_ENGINE=1 BLAST_PAIR_RESCAP=0 BLAST_PAIR_STAGES=5
