set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1; echo build $?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2f_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke $?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f_bench.log 2>&1; echo bench $?
head -c 400 gpurun_out/r2f_bench.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2f_ref.log 2>&1; echo ref $?
head -c 300 gpurun_out/r2f_ref.log
timeout 1200 python bench.py --gpus 1 --steps 300 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2f_bench300.log 2>&1; echo b300 $?
head -c 300 gpurun_out/r2f_bench300.log
