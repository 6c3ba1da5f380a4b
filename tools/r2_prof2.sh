set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "qkv_rope or argmax or rope_kv" > gpurun_out/r2g_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2g_pytest.log
timeout 900 python benchmarks/replay_ab.py --record 60 --rounds 3 --variants base,norope,plo0 --kernels > gpurun_out/r2g_replay_ab.log 2>&1; echo ab $?
cat gpurun_out/r2g_replay_ab.log | tail -60
