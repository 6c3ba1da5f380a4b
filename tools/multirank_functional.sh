# Functional (not a measurement) multi-rank bench runs with every rank on ONE GPU (gloo):
# disjoint generator / fixer placement at N = 2 and 4, and TP = 2 replicas (host sync).
export CORTEX_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 200 --warmup 5 --profile-steps 4 --concurrency 32 --no-cpu-baseline > gpurun_out/mr_disjoint2.log 2>&1; echo disjoint2 $?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --steps 200 --warmup 5 --profile-steps 4 --concurrency 16 --no-cpu-baseline > gpurun_out/mr_disjoint4.log 2>&1; echo disjoint4 $?
CORTEX_TP_HOST_SYNC=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --tp 2 --workload config5 --steps 200 --warmup 5 --profile-steps 4 --concurrency 16 --no-cpu-baseline > gpurun_out/mr_tp4.log 2>&1; echo tp4 $?
for f in mr_disjoint2 mr_disjoint4 mr_tp4; do tail -1 gpurun_out/$f.log | cut -c1-300; done
