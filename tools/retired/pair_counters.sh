# per-role wait counters of the CTA-pair engine (streamed and resident weights)
BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -c "from paper_2507_03117_b200 import build; build.build(force=True)" > /dev/null 2>&1
for rc in 0 999; do
  echo "== RESCAP=$rc"
  BLAST_PAIR_ENGINE=1 BLAST_PAIR_RESCAP=$rc BLAST_DEBUG_COUNTERS=1 timeout 120 python tools/diag_time.py 2>&1 | grep "blast dbg" | tail -2
  BLAST_PAIR_ENGINE=1 BLAST_PAIR_RESCAP=$rc BLAST_SKIP_EPILOGUE=3 BLAST_DEBUG_COUNTERS=1 timeout 120 python tools/diag_time.py 2>&1 | grep "blast dbg" | tail -2
done
python -c "from paper_2507_03117_b200 import build; build.build(force=True)" > /dev/null 2>&1
for rc in 0 999; do BLAST_PAIR_ENGINE=1 BLAST_PAIR_RESCAP=$rc timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:spmm_pair --csv python tools/diag_time.py 2>/dev/null | grep spmm_pair | tail -2 | awk -F'","' '{print substr($5,1,70), $NF}'; done
