timeout 600 python -m pytest tests/test_gpu_modes.py -q -x > gpurun_out/tm.log 2>&1
for e in 0 2 0 2; do echo "== split=$e"; BLAST_SPLIT_STAGES=$e timeout 120 python tools/diag_time.py; done
for e in 0 2; do BLAST_SPLIT_STAGES=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:spmm_tc --csv python tools/diag_time.py 2>/dev/null | grep spmm_tc | tail -2 | awk -F'","' '{print substr($5,1,70), $NF}'; done
