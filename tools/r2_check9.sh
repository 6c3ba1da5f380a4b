set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "gemm" > gpurun_out/r2m_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2m_pytest.log
bash tools/r2_l2exp.sh > gpurun_out/r2m_l2exp.log 2>&1; cat gpurun_out/r2m_l2exp.log
timeout 600 python benchmarks/gemm.py 204 512 768 > gpurun_out/r2m_gemm.jsonl 2>&1; echo gemm $?
timeout 900 python benchmarks/replay_ab.py --record 60 --rounds 3 --variants base,whole > gpurun_out/r2m_replay.log 2>&1; echo ab $?
tail -1 gpurun_out/r2m_replay.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 60 --warmup 5 --concurrency 32 --no-cpu-baseline > gpurun_out/r2m_n2.log 2>&1; echo n2 $?
tail -c 600 gpurun_out/r2m_n2.log
