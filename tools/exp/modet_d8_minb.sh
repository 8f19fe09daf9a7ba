#!/bin/bash
# ModeT backward at d = 8 (the SURVEY 8d stress config): resident-CTA bound A/B
set -e
cd "$(dirname "$0")/../.."
for mb in 1 2; do
  touch paper_2403_16526_b200/csrc/modet_tiled.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_BWD_MINB8=$mb" >/dev/null 2>&1
  echo "== MDG_BWD_MINB8=$mb"
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-pyramid --no-po --no-cfg2 \
      --no-random-field --no-slab-po 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['modet_stress'])"
done
