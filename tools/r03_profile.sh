#!/bin/bash
# Round-3 evidence pass on one B200 (run under gpurun from the repo root):
# launch list + ncu --set full of layer 0 (config 2, fp32-parity, one ~248k-token
# chunk = the bench's launch size), GEMM raster DRAM A/B, racecheck of the shipped
# CTA-pair GEMM, loader phases.
set -x
mkdir -p gpurun_out
export MFG_CFG=${MFG_CFG:-2} MFG_PREC=${MFG_PREC:-fp32} MFG_RECORDS=${MFG_RECORDS:-1260}
TAG=${TAG:-r03_config${MFG_CFG}_${MFG_PREC}}
python bench.py --steps 1 --warmup 3 --records-per-step 64 --no-cpu-baseline --no-parity --no-other-precisions --config $MFG_CFG > /dev/null 2>&1  # writes the container
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_window.py > gpurun_out/pw_$TAG.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"gemm2|attention_tc|layernorm" -c 6 -f -o gpurun_out/prof_$TAG python tools/profile_window.py >> gpurun_out/pw_$TAG.log 2>&1
TOK=$(grep -o "[0-9]* tokens" gpurun_out/pw_$TAG.log | head -1 | cut -d' ' -f1)
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep gpurun_out/launches_$TAG.csv $TAG $MFG_CFG $MFG_PREC $TOK
cp profiles/ncu_summary_$TAG.json gpurun_out/
# gpurun copies back at most 64 MiB: keep the full capture only when asked
[ -z "$KEEP_REP" ] && rm -f gpurun_out/prof_$TAG.ncu-rep
if [ -n "$RASTER" ]; then
  for G in 0 2 4 8 16; do
    MFG_GEMM_GROUP=$G timeout 300 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:gemm2 -c 4 --csv python tools/profile_window.py > gpurun_out/raster_g$G.csv 2>&1
  done
fi
if [ -n "$RACE" ]; then
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "k_chunked and fp32" > gpurun_out/racecheck_$TAG.txt 2>&1
  tail -30 gpurun_out/racecheck_$TAG.txt
fi
if [ -n "$LOADT" ]; then
  MFG_LOAD_TRACE=1 timeout 300 python tools/load_time.py $MFG_CFG > gpurun_out/load_$TAG.txt 2>&1
  cat gpurun_out/load_$TAG.txt
fi
