#!/bin/bash
# A/B an environment switch on one library: tools/ab_env.sh "VAR=a" "VAR=b" [rounds]
for i in $(seq ${3:-3}); do
  for e in "$1" "$2"; do
    env $e timeout 300 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$e', round(d['ms_per_step'],4), repr(d['loss_last']))"
  done
done
