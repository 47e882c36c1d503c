#!/bin/bash
# A/B bench with the final loss (bit-identity check): tools/ab_loss.sh "ENV_A" "ENV_B" [rounds]
for i in $(seq ${3:-2}); do
  for v in "$1" "$2"; do
    env $v timeout 300 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['ms_per_step'],4), repr(d['loss_last']))"
  done
done
