# build each -D variant on the box and print the engine's per-role cycle counters
for v in "-DBLAST_BALLOT_GU=1" "-DBLAST_BALLOT_GU=1 -DBLAST_WAITER_GU=1"; do
  echo "#### $v"
  BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS $v" python -c "from paper_2507_03117_b200 import build; build.build(force=True)" > /dev/null 2>&1
  bash tools/diag_counters.sh
done
