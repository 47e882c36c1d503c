#!/bin/bash
# Full GPU check: test suite, bench lines (bf16 default, tf32), reference arm.
set -u
tag=${1:-r02}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/gputest_$tag.log 2>&1; echo tests=$?
tail -25 gpurun_out/gputest_$tag.log
PC_BENCH_BREAKDOWN=1 timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
PC_BENCH_BREAKDOWN=1 timeout 600 python bench.py --precision tf32 --no-cpu-baseline > gpurun_out/bench_tf32_$tag.json 2> gpurun_out/bench_tf32_$tag.err; echo bench_tf32=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo ref=$?
