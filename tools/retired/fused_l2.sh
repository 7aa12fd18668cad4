# fused gate+up->down kernel: time and DRAM traffic with / without discarding consumed G slots
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x 2>&1 | tail -1
for d in 0 8; do
  echo "== BLAST_FUSED_DBG=$d"
  BLAST_FUSED_MLP=1 BLAST_FUSED_DBG=$d timeout 120 python tools/diag_time.py
  BLAST_FUSED_MLP=1 BLAST_FUSED_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:mlp_fused -c 3 --csv python tools/diag_time.py 2>/dev/null | grep mlp_fused | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
echo "== two-launch path"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:spmm_tc -c 6 --csv python tools/diag_time.py 2>/dev/null | grep spmm_tc | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
