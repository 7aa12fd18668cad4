# same-box cfg3 forward under the opt-in engine modes (no rebuilds)
run() { echo "== $*"; env "$@" timeout 300 python bench.py --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])"; }
for i in 1 2; do
  run BLAST_SPLIT_STAGES=0
  run BLAST_SPLIT_STAGES=2
  run BLAST_SPLIT_STAGES=1
done
