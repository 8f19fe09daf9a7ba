#!/bin/bash
# ncu recipe used for profiles/ (run under gpurun, 1 GPU; B200_PROFILING.md)
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:'modet_fwd_k|modet_bwd_k|warp_fwd_k|warp_bwd_k' -s 12 -c 4 \
    -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
