# Round-2 check on one B200: GPU tests, the driver's bench command, and the ncu launch
# list (time + DRAM bytes) of exactly the bench's timed steps (CORTEX_NCU_TIMED=1).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2_pytest.log 2>&1; echo pytest $?
tail -5 gpurun_out/r2_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2>&1; echo bench $?
tail -c 3000 gpurun_out/r2_bench.log
CORTEX_NCU_TIMED=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_timed.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_ncu.log 2>&1; echo ncu $?
