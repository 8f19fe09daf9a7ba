#!/bin/bash
# ModeT forward: resident-CTA bound A/B (bench per-op times)
set -e
cd "$(dirname "$0")/../.."
for mb in 3 4; do
  touch paper_2403_16526_b200/csrc/modet_tiled.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_FWD_MINB=$mb" >/dev/null 2>&1
  echo "== MDG_FWD_MINB=$mb"
  cuobjdump -res-usage paper_2403_16526_b200/libmdg.so 2>/dev/null | grep -A1 "modet_fwd_tiled_kILi6ELb1" | grep -o "REG:[0-9]* STACK:[0-9]*" | tr '\n' ' '; echo
  python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-pyramid --no-po --no-cfg2 \
      --no-random-field --no-stress --no-slab-po 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['per_op_ms'])"
done
