# same-box cfg2 training step and cfg3 forward: an older build copied to _ab_c/ vs the working tree
for i in 1 2; do
  for t in _ab_c .; do
    (cd $t && timeout 600 python tools/config_sweep.py cfg2 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$t cfg2', round(d['sparse_fwd_bwd_ms'],3), round(d['dense_fwd_bwd_ms'],3))")
    (cd $t && timeout 300 python bench.py --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$t cfg3', round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])")
  done
done
