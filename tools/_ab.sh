mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python tools/profile_window.py > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gemm2|attention_tc|layernorm" -c 6 -f -o gpurun_out/prof_r02 python tools/profile_window.py > gpurun_out/ncu_r02.log 2>&1
for P in fp16 bf16; do
MFG_PREC=$P timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_$P.csv python tools/profile_window.py > /dev/null 2>&1
done
ls -la gpurun_out
