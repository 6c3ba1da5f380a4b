# Round-1 final profile set (run under gpurun from the repo root): the bench command
# alone (must exit 0), then its launch list with DRAM bytes (-> profiles/traffic.json and
# the launch-share summary), then full captures of the step's top kernels: the 2-SM GEMM,
# the cluster split-K GEMM, the tcgen05 FMHA (two-tile) and the paged decode kernel.
set -x
B="python bench.py --steps 3 --warmup 150 --profile-steps 1 --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && echo plain-ok
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 50000 -c 1500 --csv --log-file gpurun_out/launches_dram.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_2sm<" -s 3000 -c 2 -o gpurun_out/prof_gemm2 $B > gpurun_out/ncu_g2.log 2>&1; echo ncu2 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm_splitk -s 3000 -c 2 -o gpurun_out/prof_splitk $B > gpurun_out/ncu_sk.log 2>&1; echo ncu3 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fmha|paged_decode" -s 4000 -c 6 -o gpurun_out/prof_attn $B > gpurun_out/ncu_attn.log 2>&1; echo ncu4 $?
ls -la gpurun_out
