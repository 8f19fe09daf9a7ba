#!/bin/bash
set -e
cd "$(dirname "$0")/../.."
for mb in 2 3 4; do
  touch paper_2403_16526_b200/csrc/project.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_PROJ_BWD_MINB=$mb" >/dev/null 2>&1
  echo "== MDG_PROJ_BWD_MINB=$mb"; python tools/exp/proj_bwd_time.py
done
