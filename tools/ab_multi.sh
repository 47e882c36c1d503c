#!/bin/bash
# A/B/C/... of environment settings on one library: tools/ab_multi.sh rounds "VAR=a" "VAR=b" ...
rounds=$1; shift
for i in $(seq $rounds); do
  for e in "$@"; do
    env $e timeout 300 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$e', round(d['ms_per_step'],4), repr(d['loss_last']))"
  done
done
