#!/bin/bash
# y-pair warp bwd: occupancy bound A/B at the bench workload (C = 8)
set -e
cd "$(dirname "$0")/../.."
for mb in 2; do
  touch paper_2403_16526_b200/csrc/sampling.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_PAIR_MINB=$mb" >/dev/null 2>&1
  echo "== MDG_PAIR_MINB=$mb"
  python tools/exp/warp_split.py 2>&1 | grep -E "both|gfield ms|gin    ms|C= 8|C=16|C= 1"
done
