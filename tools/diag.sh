for e in 0 1 2 3; do
# (skip modes 2/3 need the library built with BLAST_NVCC_FLAGS=-DBLAST_DIAG_SWITCHES=1)
  echo "== skip=$e"; BLAST_SKIP_EPILOGUE=$e timeout 120 python tools/diag_time.py
  BLAST_SKIP_EPILOGUE=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:spmm_tc --csv python tools/diag_time.py 2>/dev/null | grep spmm_tc | tail -2 | awk -F'","' '{print substr($5,1,60), $NF}'
done
