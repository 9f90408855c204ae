#!/bin/bash
# Dynamic (atomic-counter) vs static round-robin tile hand-out in the CTA-pair GEMM:
# same-box alternating bench runs (MFG_TILE_DYN=0 is the static schedule).
for i in 1 2; do
  for D in 0 1; do
    MFG_TILE_DYN=$D timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-parity --no-other-precisions "$@" 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dyn=$D', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
  done
done
