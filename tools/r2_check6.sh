set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x > gpurun_out/r2h_pytest.log 2>&1; echo pytest $?
tail -15 gpurun_out/r2h_pytest.log
timeout 600 python benchmarks/gemm.py 64 204 256 > gpurun_out/r2h_gemm.jsonl 2>&1; echo gemm $?
timeout 900 python benchmarks/replay_ab.py --record 60 --rounds 3 --variants base --kernels > gpurun_out/r2h_replay.log 2>&1; echo ab $?
cat gpurun_out/r2h_replay.log | tail -40
