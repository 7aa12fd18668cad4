for r in 1 2 3; do for l in base new; do echo -n "$l: "; export BLAST_LIB=$PWD/ab_libs/libblast_$l.so; python tools/config_sweep.py cfg3 64 8192 0.8,0.9,0.95 2>/dev/null | python -c "
import sys, json
print('  '.join(f'{json.loads(l)[\"sparsity\"]}: {json.loads(l)[\"sparse_ms\"]*1e3:.1f}us' for l in sys.stdin))"; done; done
unset BLAST_LIB
python -m pytest tests/test_gpu_products.py tests/test_gpu_mlp.py tests/test_gpu_modes.py tests/test_gpu_configs.py -q -x 2>&1 | tail -1
