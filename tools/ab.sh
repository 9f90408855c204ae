#!/bin/bash
# Same-box A/B of two libmfgpu builds (lib/libmfgpu_base.so vs lib/libmfgpu.so):
# alternating bench runs, device value + attention class time/share.
#   bash tools/ab.sh [extra bench args...]
for i in 1 2; do
  for L in libmfgpu_base.so libmfgpu.so; do
    MFG_GPU_LIB=$L timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-parity --no-other-precisions "$@" 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$L', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], 'att share', round(r['class_ms_share']['attention'],4), 'att frac', round(r.get('attention_hbm',{}).get('frac',0),3))"
  done
done
