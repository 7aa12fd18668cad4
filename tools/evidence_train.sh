#!/bin/bash
# ncu --set full of the cfg3 training-step kernels changed late in round 2: the gating backward
# (dG, 3rd spmm_tc launch of the 4th iteration) and the first weight gradient (dWdown) of the
# same iteration; tools/extras_once.py train. Outputs under gpurun_out/r02_train/.
set -u
O=gpurun_out/r02_train
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_tc -s 14 -c 1 -o $O/full_dgrad -f python tools/extras_once.py train > $O/ncu_dgrad.log 2>&1
tail -1 $O/ncu_dgrad.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wgrad_tc -s 9 -c 1 -o $O/full_wgrad -f python tools/extras_once.py train > $O/ncu_wgrad.log 2>&1
tail -1 $O/ncu_wgrad.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_train.csv python tools/extras_once.py train > /dev/null 2>&1
python tools/ncu_summary.py $O/full_dgrad.ncu-rep > $O/summary_dgrad.txt 2>&1
python tools/ncu_summary.py $O/full_wgrad.ncu-rep > $O/summary_wgrad.txt 2>&1
cat $O/summary_dgrad.txt $O/summary_wgrad.txt
