set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2p_build.log 2>&1; echo build $?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2p_pytest.log 2>&1; echo pytest $?
tail -4 gpurun_out/r2p_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2p_bench.log 2>&1; echo bench $?
head -c 600 gpurun_out/r2p_bench.log
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2p_launches_timed.csv python bench.py --gpus 1 --steps 3 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2p_ncu.log 2>&1; echo ncu $?
cp gpurun_out/ncu_window_algorithmic.json gpurun_out/r2p_ncu_window_algorithmic.json
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"gemm_bf16_2sm<" -c 2 -o gpurun_out/r2p_ncu_gemm2_step python bench.py --gpus 1 --steps 2 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2p_ncu_full.log 2>&1; echo ncufull $?
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"paged_decode_kernel" -c 2 -o gpurun_out/r2p_ncu_decode_step python bench.py --gpus 1 --steps 2 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2p_ncu_full2.log 2>&1; echo ncufull2 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 60 --warmup 5 --concurrency 32 --no-cpu-baseline > gpurun_out/r2p_n2.log 2>&1; echo n2 $?
tail -c 400 gpurun_out/r2p_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --tp 2 --steps 30 --warmup 5 --concurrency 16 --workload config5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2p_tp2.log 2>&1; echo tp2 $?
tail -c 400 gpurun_out/r2p_tp2.log
