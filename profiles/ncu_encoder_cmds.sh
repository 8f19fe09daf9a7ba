#!/bin/bash
# ncu recipe for the encoder conv kernels at the L0 shape of 160x192x224
# (8 -> 8 channels): fwd (conv3t_k), kernel gradient (conv3w_k), and the deep
# level's implicit GEMM (L3 64 -> 64).  One GPU, after the plain run exits 0.
set -e
ONLY=L0:8:8 python tools/bench_conv.py > gpurun_out/conv_plain.log 2>&1
ONLY=L0:8:8 ncu --set full --clock-control none --import-source on -k regex:conv3t_k \
    -c 1 -o gpurun_out/enc_l0 python tools/bench_conv.py > gpurun_out/ncu_enc_l0.log 2>&1
ONLY=L0:8:8 ncu --set full --clock-control none --import-source on -k regex:conv3w_k \
    -c 1 -o gpurun_out/enc_l0w python tools/bench_conv.py > gpurun_out/ncu_enc_l0w.log 2>&1
ONLY=L3:64:64 ncu --set full --clock-control none --import-source on -k regex:igemm_fwd \
    -c 1 -o gpurun_out/enc_l3 python tools/bench_conv.py > gpurun_out/ncu_enc_l3.log 2>&1
echo "ncu encoder rc=0"
