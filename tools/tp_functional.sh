# Functional (not a measurement) TP=2 bench runs with every rank on ONE GPU: gloo process
# group, host barrier at every exchange point (CORTEX_TP_HOST_SYNC), so no kernel spins on another rank.
export CORTEX_DIST_BACKEND=gloo CORTEX_TP_HOST_SYNC=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --tp 2 --placement replicas --steps 300 --warmup 5 --profile-steps 4 --concurrency 16 --no-cpu-baseline > gpurun_out/tp_bench2.log 2>&1; echo tpbench2 $?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --tp 2 --workload config5 --steps 300 --warmup 5 --profile-steps 4 --concurrency 16 --no-cpu-baseline > gpurun_out/tp_bench4.log 2>&1; echo tpbench4 $?
tail -3 gpurun_out/tp_bench2.log; tail -3 gpurun_out/tp_bench4.log
