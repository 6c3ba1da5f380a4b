set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1; echo build $?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2w_pytest.log 2>&1; echo pytest $?
tail -4 gpurun_out/r2w_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2w_bench.log 2>&1; echo bench $?
head -c 400 gpurun_out/r2w_bench.log
timeout 600 python benchmarks/host_overhead.py > gpurun_out/r2w_host.log 2>&1; echo host $?
tail -2 gpurun_out/r2w_host.log
