#!/bin/bash
# ModeT backward row / column kernels: resident-CTA bound A/B (bench per-op times)
set -e
cd "$(dirname "$0")/../.."
for mb in 2 3; do
  touch paper_2403_16526_b200/csrc/modet_tiled.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_BWD_MINB=$mb" >/dev/null 2>&1
  echo "== MDG_BWD_MINB=$mb"
  python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-pyramid --no-po --no-cfg2 \
      --no-random-field 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['per_op_ms'], d['modet_stress'])"
done
