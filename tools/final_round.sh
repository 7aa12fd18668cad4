# Round-end evidence on one GPU box: tests, bench line, launch list, ncu full capture of the
# two MLP kernels, graph replay, cfg2 training step. Outputs under gpurun_out/final/.
set -u
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1200 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dense > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:spmm_tc -s 2 -c 2 -o $O/full_cfg3 python tools/prof_once.py > $O/ncu_full.log 2>&1
timeout 300 python tools/graph_probe.py > $O/graph_probe.txt 2>&1
timeout 900 python tools/config_sweep.py cfg2 > $O/cfg2.jsonl 2> $O/cfg2.err
