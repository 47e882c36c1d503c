#!/bin/bash
# A/B two prebuilt libraries: tools/ab_lib.sh libA.so libB.so [rounds]
for i in $(seq ${3:-3}); do
  for lib in "$1" "$2"; do
    cp "$lib" paper_1312_5853_b200/libpcb200.so
    timeout 300 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', round(d['ms_per_step'],4), repr(d['loss_last']))"
  done
done
