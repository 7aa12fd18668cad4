#!/bin/bash
# Same-box A/B of an environment switch on the cfg3 forward (tools/diag_time.py), alternating
# runs: tools/ab_env.sh VAR VALUE_A VALUE_B [sparsity]
var=$1; a=$2; b=$3; sp=${4:-0.9}
for i in 1 2 3; do
  for v in $a $b; do
    echo -n "$var=$v: "; env $var=$v python tools/diag_time.py $sp
  done
done
