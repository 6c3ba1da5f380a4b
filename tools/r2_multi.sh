mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 60 --warmup 5 --concurrency 32 --no-cpu-baseline > gpurun_out/r2m2_n2.log 2>&1; echo n2 $?
tail -c 300 gpurun_out/r2m2_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --mode shared --steps 60 --warmup 5 --concurrency 32 --no-cpu-baseline --no-shared-arm > gpurun_out/r2m2_n2s.log 2>&1; echo n2s $?
tail -c 300 gpurun_out/r2m2_n2s.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus 2 --tp 2 --steps 30 --warmup 5 --concurrency 16 --workload config5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2m2_tp2.log 2>&1; echo tp2 $?
tail -c 300 gpurun_out/r2m2_tp2.log
