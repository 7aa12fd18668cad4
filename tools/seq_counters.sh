BLAST_NVCC_FLAGS="-DBLAST_WAIT_COUNTERS" python -c "from paper_2507_03117_b200 import build; build.build(force=True)" > /dev/null 2>&1
for m in 0 2; do echo "#### split=$m"; BLAST_SPLIT_STAGES=$m bash tools/diag_counters.sh; done
