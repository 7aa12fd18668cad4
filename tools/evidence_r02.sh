#!/bin/bash
# Round-2 evidence on one GPU box: tests, smoke, bench line, launch list of the bench command,
# ncu --set full of the two cfg3 forward kernels. Outputs under gpurun_out/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dense --no-extras > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:spmm_tc -s 2 -c 2 -o $O/full_cfg3 -f python tools/prof_once.py > $O/ncu_full.log 2>&1
tail -1 $O/ncu_full.log
