set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo build $?
for s in "512 6144 4096" "768 6144 4096" "204 28672 4096" "700 4096 4096"; do timeout 60 python tools/one_gemm.py $s 2>&1 | tail -1; done
timeout 1200 python -m pytest tests/test_kernels_gpu.py -q -m gpu > gpurun_out/r2o_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2o_pytest.log
timeout 900 python benchmarks/replay_ab.py --record 60 --rounds 2 --variants base > gpurun_out/r2o_replay.log 2>&1; echo ab $?
tail -1 gpurun_out/r2o_replay.log
