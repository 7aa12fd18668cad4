timeout 900 python -m pytest tests/test_gpu_modes.py -q -x 2>&1 | tail -1
bash tools/ab_bench.sh
