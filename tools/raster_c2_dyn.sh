#!/bin/bash
# Raster re-check with the dynamic tile hand-out: config-2 layer-0 GEMM DRAM bytes per MFG_GEMM_GROUP.
export MFG_CFG=2 MFG_RECORDS=1260
python bench.py --steps 1 --warmup 3 --records-per-step 64 --no-cpu-baseline --no-parity --no-other-precisions > /dev/null 2>&1
for G in 0 2 4 8; do
  MFG_GEMM_GROUP=$G timeout 300 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm2 -c 4 --csv python tools/profile_window.py > gpurun_out/rdyn_g$G.csv 2>&1
done
