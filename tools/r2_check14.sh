set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1; echo build $?
timeout 600 python -m pytest tests/test_step_gpu.py -q -x > gpurun_out/r2x_step.log 2>&1; echo step $?
tail -15 gpurun_out/r2x_step.log
timeout 600 python benchmarks/host_overhead.py > gpurun_out/r2x_host.log 2>&1; echo host $?
tail -2 gpurun_out/r2x_host.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2x_bench.log 2>&1; echo bench $?
head -c 500 gpurun_out/r2x_bench.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2x_pytest.log 2>&1; echo pytest $?
tail -4 gpurun_out/r2x_pytest.log
