# same-box cfg3: single-buffered output staging for the single-matrix products (_ab_ob) vs default
(cd _ab_ob && timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_gpu_modes.py -q -x 2>&1 | tail -1)
for i in 1 2; do
  for t in _ab_ob .; do
    (cd $t && timeout 300 python bench.py --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$t', round(d['ms_per_step'],4), d['mlp_roofline']['kernel_ms'])")
  done
done
