set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1; echo build $?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2i_pytest.log 2>&1; echo pytest $?
tail -15 gpurun_out/r2i_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2i_bench.log 2>&1; echo bench $?
head -c 1200 gpurun_out/r2i_bench.log
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2i_launches_timed.csv python bench.py --gpus 1 --steps 3 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2i_ncu.log 2>&1; echo ncu $?
tail -3 gpurun_out/r2i_ncu.log
