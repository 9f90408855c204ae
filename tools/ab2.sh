#!/bin/bash
# Same-box A/B of two libmfgpu builds given by name (in lib/): bash tools/ab2.sh A.so B.so [bench args...]
A=$1; B=$2; shift 2
for i in 1 2; do
  for L in $A $B; do
    MFG_GPU_LIB=$L timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-parity --no-other-precisions "$@" 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$L', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], {k: round(v,4) for k,v in r['class_ms_share'].items() if k in ('qkv','o_proj','ffn1','ffn2','attention','layernorm')})"
  done
done
