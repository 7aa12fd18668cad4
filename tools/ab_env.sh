#!/bin/bash
# Same-box A/B of an engine environment switch on the decode extra and the cfg3 bench:
#   bash tools/ab_env.sh VAR        (runs VAR=1 and VAR=0 alternately, three rounds)
v=$1
for r in 1 2 3; do for x in 1 0; do
  echo -n "$v=$x decode: "; env $v=$x python tools/extras_quick.py decode | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['us'],2), 'us')"
done; done
