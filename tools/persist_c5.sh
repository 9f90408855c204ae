#!/bin/bash
# L2-persisting window for the K-chunk partial buffer: config-5 layer-0 GEMM DRAM
# bytes with and without (MFG_L2_PERSIST=0), then same-box bench A/B.
export MFG_CFG=5 MFG_RECORDS=3700
python bench.py --steps 1 --warmup 3 --records-per-step 64 --no-cpu-baseline --no-parity --no-other-precisions --config 5 > /dev/null 2>&1
for P in 0 1; do
  MFG_L2_PERSIST=$P timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm2 -c 4 --csv python tools/profile_window.py > gpurun_out/persist_c5_p$P.csv 2>&1
done
for P in 0 1 0 1; do
  MFG_L2_PERSIST=$P timeout 900 python bench.py --config 5 --steps 10 --records-per-step 1000 --no-cpu-baseline --no-parity --no-other-precisions 2>/dev/null \
  | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('persist=$P', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], 'att share', round(r['class_ms_share']['attention'],4), 'att frac', round(r.get('attention_hbm',{}).get('frac',0),3))"
done
