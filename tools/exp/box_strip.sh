#!/bin/bash
# NCC box sums: outputs per thread along the summed axis (kStrip) A/B
set -e
cd "$(dirname "$0")/../.."
for k in 4 8 16; do
  touch paper_2403_16526_b200/csrc/loss.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_BOX_STRIP=$k" >/dev/null 2>&1
  echo "== kStrip $k"
  PROFILE=1 python tools/prof_loss.py 2>/dev/null | grep -E "loss fwd|box" | tail -7
done
