#!/bin/bash
# ncu recipe for profiles/ (run under gpurun, 1 GPU; B200_PROFILING.md).
#   usage: bash profiles/ncu_cmds.sh <tag>
# 1. the bench step runs plain first (must exit 0);
# 2. launch list of the bench step with per-launch time + DRAM bytes (every
#    kernel of the timed steps, incl. modet_bwd_row_k / modet_bwd_col_k);
# 3. --set full of each of the step's kernels, one launch each, after warm-up;
# 4. every kernel of one PO iteration (encoder, pyramid, projection, ModeT,
#    warps, loss, Adam) with time + DRAM bytes (tools/po_iter_once.py).
# Summarise here with: python profiles/summarize_ncu.py <tag>
TAG=${1:-r02}
O=gpurun_out/ncu_$TAG
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pyramid --no-po --no-cfg2 --no-random-field --no-stress --no-slab-po"
$CMD > $O/plain.log 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --metrics $M --clock-control none --csv --log-file $O/step_launches.csv $CMD > $O/step.log 2>&1
# full captures are large: keep the raw-metric CSV of each (what the summary
# reads) and the .ncu-rep only for KEEP_REPS kernels (gpurun returns <= 64 MiB)
for K in modet_fwd_tiled_k modet_bwd_row_k modet_bwd_col_k warp_fwd_k warp_bwd_k; do
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 3 -c 1 \
      -o $O/full_$K $CMD > $O/full_$K.log 2>&1
  ncu -i $O/full_$K.ncu-rep --page raw --csv > $O/full_$K.raw.csv 2>/dev/null
  case " $KEEP_REPS " in *" $K "*) ;; *) rm -f $O/full_$K.ncu-rep ;; esac
done
ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file $O/po_launches.csv python tools/po_iter_once.py > $O/po.log 2>&1
# 5. --set full of one tcgen05 encoder convolution launch of the PO iteration
#    (SASS: UTCHMMA/UTCBAR; tensor-pipe utilisation)
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"conv_k" -c 1 -o $O/full_tc_conv_k python tools/po_iter_once.py > $O/full_tc_conv_k.log 2>&1
ncu -i $O/full_tc_conv_k.ncu-rep --page raw --csv > $O/full_tc_conv_k.raw.csv 2>/dev/null
echo "ncu rc=$?"
