#!/bin/bash
# The bench line for every BASELINE config (fp32-parity) plus config 2 in the
# reference fp16 mode; JSON lines into gpurun_out/bench_r03_config<N>[_prec].log
for C in ${CONFIGS:-1 3 4 5}; do
  timeout 1500 python bench.py --config $C > gpurun_out/bench_r03_config$C.log 2> gpurun_out/bench_r03_config$C.err
  tail -c 300 gpurun_out/bench_r03_config$C.log
done
if [ -n "$FP16" ]; then
  timeout 900 python bench.py --precision fp16 --no-other-precisions > gpurun_out/bench_r03_config2_fp16.log 2> gpurun_out/bench_r03_config2_fp16.err
  tail -c 300 gpurun_out/bench_r03_config2_fp16.log
fi
