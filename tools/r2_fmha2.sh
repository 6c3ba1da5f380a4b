set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "attention or fmha or cascade" > gpurun_out/r2k_pytest.log 2>&1; echo pytest $?
tail -5 gpurun_out/r2k_pytest.log
timeout 300 python benchmarks/attn_step.py > gpurun_out/r2k_attn_step.log 2>&1; echo attn $?
tail -2 gpurun_out/r2k_attn_step.log
timeout 900 python benchmarks/replay_ab.py --record 60 --rounds 3 --variants base,fmha1q,fmha2q > gpurun_out/r2k_replay.log 2>&1; echo ab $?
tail -2 gpurun_out/r2k_replay.log
