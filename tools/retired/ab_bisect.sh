# same-box cfg3 forward: previous good build vs the working tree (default and -DBLAST_DYN_QUEUE=1 copies)
for i in 1 2; do
  for t in _ab_ks .; do
    (cd $t && timeout 300 python bench.py --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$t', round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])")
  done
done
