# A/B of kernel variants on a fixed step mix, live step timeline (CUPTI), TP test re-run,
# full ncu captures of the 2-SM GEMM at mixed-step M
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1; echo build $?
timeout 600 python -m pytest tests/test_tp_gpu.py -q -m gpu > gpurun_out/r2f_tp.log 2>&1; echo tp $?
tail -3 gpurun_out/r2f_tp.log
timeout 900 python benchmarks/replay_ab.py --record 60 --rounds 3 --variants base,plo0,norope,logits > gpurun_out/r2f_replay_ab.log 2>&1; echo ab $?
tail -3 gpurun_out/r2f_replay_ab.log
timeout 900 python benchmarks/step_trace.py --steps 30 --warmup 20 --json gpurun_out/r2f_step_trace.json > gpurun_out/r2f_step_trace.log 2>&1; echo trace $?
tail -40 gpurun_out/r2f_step_trace.log
for spec in "gate_up 512" "down 512" "qkv 768"; do
  set -- $spec
  timeout 300 python benchmarks/gemm_one.py $1 $2 > /dev/null 2>&1 || echo "plain run failed $1 $2"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_2sm -s 2 -c 1 -o gpurun_out/r2f_ncu_g2_$1_$2 python benchmarks/gemm_one.py $1 $2 > gpurun_out/r2f_ncu_g2_$1_$2.log 2>&1; echo ncu $1 $2 $?
done
ls gpurun_out/*.ncu-rep
