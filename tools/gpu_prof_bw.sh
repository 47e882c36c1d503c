#!/bin/bash
# ncu --set full on the bandwidth kernels of one AlexNet step (second, eager step),
# plus the LRN + dropout net bench line.
set -u
tag=${1:-r02}
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"maxpool|s2d|softmax|sgd_k|reduce_partials|colsum|pool_bias|lrn|dropout|fc_reduce" \
  --launch-skip 16 --launch-count 20 -o gpurun_out/prof_bw_$tag python tools/prof_step_once.py > gpurun_out/prof_bw_$tag.log 2>&1; echo ncu_bw=$?
PC_BENCH_BREAKDOWN=1 timeout 600 python bench.py --net configs/alexnet_lrn_dropout.net --no-cpu-baseline > gpurun_out/bench_lrn_$tag.json 2> gpurun_out/bench_lrn_$tag.err; echo bench_lrn=$?
tail -3 gpurun_out/bench_lrn_$tag.err
