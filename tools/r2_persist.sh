mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1; echo build $?
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "persistent or paged_decode or cascade" > gpurun_out/r2t_pytest.log 2>&1; echo pytest $?
tail -4 gpurun_out/r2t_pytest.log
for r in 1 2; do
for kn in DECODE_PERSIST=0 DECODE_PERSIST=1; do
  for sc in 1 2; do
    CORTEX_KNOBS=$kn CORTEX_PRIV_SCALE=$sc timeout 300 python benchmarks/attn_step.py --private-only
  done
done
done
