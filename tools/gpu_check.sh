#!/bin/bash
# One GPU call: GPU test suite, bench line (+ per-kernel breakdown), ncu launch list of
# one step with DRAM bytes per launch (bandwidth-kernel evidence).
set -u
tag=${1:-r02}
tests=${2:-1}
if [ "$tests" = "1" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/gputest_$tag.log 2>&1; echo tests=$?
  tail -30 gpurun_out/gputest_$tag.log
fi
PC_BENCH_BREAKDOWN=1 timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
head -c 1500 gpurun_out/bench_$tag.json; echo; tail -45 gpurun_out/bench_$tag.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_launch_$tag.log 2>&1; echo ncu_launch=$?
