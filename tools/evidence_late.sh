#!/bin/bash
# Late round-2 evidence on one GPU box: smoke, bench line, launch list of the bench command,
# ncu --set full of the two cfg3 forward kernels and of the decode pair. Outputs: gpurun_out/late/.
set -u
O=gpurun_out/late
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dense > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:spmm_tc -s 2 -c 2 -o $O/full_cfg3 -f python tools/prof_once.py > $O/ncu_full.log 2>&1
tail -1 $O/ncu_full.log
python tools/ncu_summary.py $O/full_cfg3.ncu-rep > $O/ncu_full_cfg3_summary.txt 2>&1
timeout 300 python tools/graph_probe.py > $O/graph_probe.txt 2>&1; cat $O/graph_probe.txt
