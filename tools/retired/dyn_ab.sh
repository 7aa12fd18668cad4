# dynamic item queue: correctness (full GPU suite with it on) and cfg3 A/B on one box
BLAST_DYN_ITEMS=1 timeout 300 python tools/diag_time.py || echo "DYN SMOKE FAILED"
BLAST_DYN_ITEMS=1 timeout 1200 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
run() { echo "== $*"; env "$@" timeout 300 python bench.py --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])"; }
run BLAST_DYN_ITEMS=0
run BLAST_DYN_ITEMS=1
run BLAST_DYN_ITEMS=0
run BLAST_DYN_ITEMS=1
for e in 0 1; do BLAST_DYN_ITEMS=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:spmm_tc --csv python tools/diag_time.py 2>/dev/null | grep spmm_tc | tail -2 | awk -F'","' '{print substr($5,1,70), $NF}'; done
