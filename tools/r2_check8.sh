set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1; echo build $?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2l_pytest.log 2>&1; echo pytest $?
tail -4 gpurun_out/r2l_pytest.log
timeout 900 python bench.py --gpus 1 --steps 300 --warmup 5 --no-shared-arm --no-cpu-baseline > gpurun_out/r2l_bench300.log 2>&1; echo bench300 $?
head -c 700 gpurun_out/r2l_bench300.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 100 --warmup 5 --concurrency 64 --no-cpu-baseline > gpurun_out/r2l_bench_n2_func.log 2>&1; echo n2 $?
tail -c 1500 gpurun_out/r2l_bench_n2_func.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 60 --warmup 5 --concurrency 32 --split 1:3 --workload config5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2l_bench_n4_c5_func.log 2>&1; echo n4 $?
tail -c 1500 gpurun_out/r2l_bench_n4_c5_func.log
