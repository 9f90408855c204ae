#!/bin/bash
# GEMM raster experiment at config 5 (XLM-R XL: weights 79-105 MB per GEMM, larger than
# what stays L2-resident under the activation streams): layer-0 GEMM DRAM bytes + time
# per MFG_GEMM_GROUP, then same-box bench A/B.
export MFG_CFG=5 MFG_RECORDS=3700
python bench.py --steps 1 --warmup 3 --records-per-step 64 --no-cpu-baseline --no-parity --no-other-precisions --config 5 > /dev/null 2>&1
for G in 0 8 16 32; do
  MFG_GEMM_GROUP=$G timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm2 -c 4 --csv python tools/profile_window.py > gpurun_out/raster_c5_g$G.csv 2>&1
done
for G in 0 16 0 16; do
  MFG_GEMM_GROUP=$G timeout 900 python bench.py --config 5 --steps 10 --records-per-step 1000 --no-cpu-baseline --no-parity --no-other-precisions 2>/dev/null \
  | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('G=$G', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
