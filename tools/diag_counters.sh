# per-role cycle counters (library built with -DBLAST_WAIT_COUNTERS), normal and skip-all
for e in 0 3; do
  echo "== skip=$e"; BLAST_DEBUG_COUNTERS=1 BLAST_SKIP_EPILOGUE=$e timeout 120 python tools/diag_time.py 2>&1 | grep "blast dbg" | tail -4
done
