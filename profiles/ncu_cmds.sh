#!/bin/bash
# ncu recipe used for profiles/ (run under gpurun, 1 GPU; B200_PROFILING.md)
# usage: bash profiles/ncu_cmds.sh '<kernel regex>' <skip> <count>
RX=${1:-'modet|warp_fwd_k|warp_bwd_k'}
SKIP=${2:-15}
CNT=${3:-5}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pyramid --no-po"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"$RX" -s $SKIP -c $CNT \
    -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
