set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q_build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "cascade or attention" > gpurun_out/r2q_attn.log 2>&1; echo attn $?
tail -4 gpurun_out/r2q_attn.log
timeout 900 python benchmarks/replay_ab.py --record 60 --rounds 3 --variants base,nofuse > gpurun_out/r2q_replay.log 2>&1; echo ab $?
tail -6 gpurun_out/r2q_replay.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2q_pytest.log 2>&1; echo pytest $?
tail -4 gpurun_out/r2q_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2q_bench.log 2>&1; echo bench $?
head -c 600 gpurun_out/r2q_bench.log
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"gemm_bf16_2sm$" -c 2 -o gpurun_out/r2q_ncu_gemm2_step python bench.py --gpus 1 --steps 2 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2q_ncu_full.log 2>&1; echo ncufull $?
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"gemm_bf16_2sm_splitk" -c 2 -o gpurun_out/r2q_ncu_splitk_step python bench.py --gpus 1 --steps 2 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2q_ncu_full2.log 2>&1; echo ncufull2 $?
ls gpurun_out/*.ncu-rep
