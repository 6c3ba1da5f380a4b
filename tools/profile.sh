# Round profiling recipe (run under gpurun from the repo root).
set -x
B="python bench.py --steps 3 --warmup 150 --profile-steps 1 --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && echo plain-ok && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 50000 -c 1200 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
ncu --set full --clock-control none --import-source on -k regex:paged_prefill -s 2000 -c 2 -o gpurun_out/prof_prefill $B > gpurun_out/ncu_prefill.log 2>&1; echo ncu2 $?
ncu --set full --clock-control none --import-source on -k regex:"cascade|paged_decode" -s 3000 -c 2 -o gpurun_out/prof_dec $B > gpurun_out/ncu_dec.log 2>&1; echo ncu3 $?
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 6000 -c 4 -o gpurun_out/prof_gemm2 $B > gpurun_out/ncu_gemm2.log 2>&1; echo ncu4 $?
ls -la gpurun_out
