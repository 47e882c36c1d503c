#!/bin/bash
# A/B bench: tools/ab.sh "ENV_A" "ENV_B" [rounds] -> ms/step per run, alternating
ra=${3:-3}
for i in $(seq $ra); do
  for v in "$1" "$2"; do
    ms=$(env $v timeout 300 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.readline())['ms_per_step'],4))")
    echo "$v $ms"
  done
done
