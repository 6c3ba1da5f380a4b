set -x
B="python bench.py --steps 3 --warmup 150 --profile-steps 1 --no-cpu-baseline"
timeout -k 5 300 $B > gpurun_out/plain.log 2>&1 && echo plain-ok && \
timeout -k 5 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 50000 -c 1200 --csv --log-file gpurun_out/launches2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
timeout -k 5 600 ncu --set full --clock-control none --import-source on -k regex:"fmha|paged_decode|decode_combine" -s 3000 -c 6 -o gpurun_out/prof_attn2 $B > gpurun_out/ncu_attn2.log 2>&1; echo ncu2 $?
