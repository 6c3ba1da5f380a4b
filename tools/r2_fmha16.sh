mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "prefill or cascade" > gpurun_out/r2d_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/r2d_pytest.log
: > gpurun_out/r2d_fmha.jsonl
for kn in FMHA_2Q=-1 FMHA_2Q=0 FMHA_2Q=1; do
  CORTEX_KNOBS=$kn timeout 120 python benchmarks/attn_step.py --fmha-only >> gpurun_out/r2d_fmha.jsonl 2>&1
done
cat gpurun_out/r2d_fmha.jsonl
