# Live step trace (torch.profiler) + one-step ncu launch list with DRAM bytes per launch.
set -x
timeout 600 python benchmarks/step_trace.py --steps 20 --json gpurun_out/step_trace.json > gpurun_out/step_trace.log 2>&1; echo trace $?
B="python bench.py --steps 3 --warmup 150 --profile-steps 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 50000 -c 800 --csv --log-file gpurun_out/launches_dram.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu $?
