#!/bin/bash
# ModeT backward: resident-CTA bound of the row and column kernels separately
set -e
cd "$(dirname "$0")/../.."
for v in "2 2" "2 3" "3 2"; do
  set -- $v
  touch paper_2403_16526_b200/csrc/modet_tiled.cu
  make -s -C paper_2403_16526_b200/csrc EXTRA="-DMDG_BWD_ROW_MINB=$1 -DMDG_BWD_COL_MINB=$2" >/dev/null 2>&1
  echo "== row $1 col $2"
  cuobjdump -res-usage paper_2403_16526_b200/libmdg.so 2>/dev/null | grep -A1 "modet_bwd_\(row\|col\)_kILi6ELb1ELb0" | grep -o "REG:[0-9]* STACK:[0-9]*" | tr '\n' ' '; echo
  python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-pyramid --no-po --no-cfg2 \
      --no-random-field --no-stress --no-slab-po 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['per_op_ms'])"
done
