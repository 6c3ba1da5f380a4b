set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1; echo build $?
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2e_pytest.log 2>&1; echo pytest $?
tail -25 gpurun_out/r2e_pytest.log
timeout 900 python bench.py --gpus 1 --steps 200 --warmup 5 --no-shared-arm --no-cpu-baseline > gpurun_out/r2e_bench.log 2>&1; echo bench $?
head -c 1500 gpurun_out/r2e_bench.log
