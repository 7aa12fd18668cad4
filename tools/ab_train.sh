#!/bin/bash
# Same-box A/B of library builds on the cfg3 training step: bash tools/ab_train.sh [lib ...]
for r in 1 2 3; do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset BLAST_LIB; else export BLAST_LIB=$PWD/$lib; fi
    echo -n "$lib: "
    python tools/extras_quick.py train | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],4), 'ms')"
  done
done
