#!/bin/bash
# A/B of warp_bwd_k occupancy bounds for CT=3/8/16 (spills vs occupancy), PO iteration per-kernel times.
set -e
cd "$(dirname "$0")/../.."
for v in "5 4" "4 3" "4 4" "3 3"; do
  set -- $v
  touch paper_2403_16526_b200/csrc/sampling.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_WBWD_MINB=$1 -DMDG_WBWD_MINB16=$2" >/dev/null
  echo "== MINB=$1 MINB16=$2"
  python tools/prof_po.py | grep -E "warp_bwd|total"
done
