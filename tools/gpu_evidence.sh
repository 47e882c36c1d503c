#!/bin/bash
# Round evidence: GPU tests, bench lines (bf16 default, tf32, LRN+dropout net),
# reference arm, ncu launch list with DRAM bytes of one step, ncu --set full of
# the dominant GEMMs (conv2 forward / data gradient / weight gradient, conv1).
set -u
tag=${1:-r02}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/gputest_$tag.log 2>&1; echo tests=$?
tail -4 gpurun_out/gputest_$tag.log
PC_BENCH_BREAKDOWN=1 timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
PC_BENCH_BREAKDOWN=1 timeout 600 python bench.py --precision tf32 --no-cpu-baseline > gpurun_out/bench_tf32_$tag.json 2> gpurun_out/bench_tf32_$tag.err; echo bench_tf32=$?
PC_BENCH_BREAKDOWN=1 timeout 600 python bench.py --net configs/alexnet_lrn_dropout.net --no-cpu-baseline > gpurun_out/bench_lrn_$tag.json 2> gpurun_out/bench_lrn_$tag.err; echo bench_lrn=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__cycles_active.avg --clock-control none --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_launch_$tag.log 2>&1; echo ncu_launch=$?
for L in L3 L0; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:umma_gemm -c 4 \
    -o gpurun_out/prof_${L}_$tag python tools/prof_conv.py $L 1 > gpurun_out/ncu_full_${L}_$tag.log 2>&1; echo ncu_$L=$?
done
