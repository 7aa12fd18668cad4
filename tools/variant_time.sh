# build each -D variant on the box; cfg3 forward time and per-kernel launch times
for v in "$@"; do
  echo "#### [$v]"
  BLAST_NVCC_FLAGS="$v" python -c "from paper_2507_03117_b200 import build; build.build(force=True)" > /dev/null 2>&1 || echo BUILD FAILED
  timeout 120 python tools/diag_time.py; timeout 120 python tools/diag_time.py
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:spmm_tc --csv python tools/diag_time.py 2>/dev/null | grep spmm_tc | tail -2 | awk -F'","' '{print substr($5,1,60), $NF}'
done
