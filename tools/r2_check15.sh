set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1; echo build $?
timeout 1200 python bench.py --gpus 1 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench300.log 2>&1; echo b300 $?
head -c 300 gpurun_out/r2c_bench300.log
timeout 1500 python bench.py --gpus 1 --steps 100 --warmup 5 --workload config4 --no-cpu-baseline --no-shared-arm > gpurun_out/r2c_config4.log 2>&1; echo c4 $?
head -c 300 gpurun_out/r2c_config4.log
timeout 1200 python bench.py --gpus 1 --steps 200 --warmup 5 --workload config5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2c_config5.log 2>&1; echo c5 $?
head -c 300 gpurun_out/r2c_config5.log
