#!/bin/bash
# One GPU call that regenerates the round's measurement artefacts under gpurun_out/:
# bench line, reference-arm line, per-kernel breakdown, ncu launch list of one
# step, and ncu --set full captures of the dominant convolution kernels.
set -u
tag=${1:-v4}
timeout 400 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>&1; echo ref=$?
PC_BENCH_BREAKDOWN=1 timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_bd_$tag.log 2>&1; echo bd=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_launch_$tag.log 2>&1; echo ncu_launch=$?
for L in L3 L0; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:umma_gemm -c 6 \
    -o gpurun_out/prof_${L}_$tag python tools/prof_conv.py $L 1 > gpurun_out/ncu_full_${L}_$tag.log 2>&1; echo ncu_$L=$?
done
