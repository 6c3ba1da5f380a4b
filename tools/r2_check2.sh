# Round-2 check #2: GPU tests, the driver's bench command, GEMM shapes of the mixed
# steps vs cuBLAS, and the ncu launch list (time + DRAM bytes) of the bench's timed steps.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1; echo build $?
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r2b_pytest.log 2>&1; echo pytest $?
tail -15 gpurun_out/r2b_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_bench.log 2>&1; echo bench $?
tail -c 4000 gpurun_out/r2b_bench.log
timeout 600 python benchmarks/gemm.py 256 512 768 1024 2048 3584 > gpurun_out/r2b_gemm.jsonl 2>&1; echo gemm $?
CORTEX_NCU_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_timed.csv python bench.py --gpus 1 --steps 3 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2b_ncu.log 2>&1; echo ncu $?
