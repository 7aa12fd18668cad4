(cd _ab_ks && timeout 600 python -m pytest ../tests/test_gpu_mlp.py -q -x -m gpu 2>&1 | tail -1) 
bash tools/ab_bisect.sh
