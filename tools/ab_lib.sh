#!/bin/bash
# Same-box A/B of library builds on the cfg3 bench (no extras): bash tools/ab_lib.sh [lib ...]
# ("default" = the in-tree build). Three alternating rounds.
for r in 1 2 3; do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset BLAST_LIB; else export BLAST_LIB=$PWD/$lib; fi
    echo -n "$lib: "
    python bench.py --steps 30 --warmup 5 --no-extras --no-cpu --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'ms', {k: round(v,4) for k,v in d['mlp_roofline']['kernel_ms'].items()})"
  done
done
