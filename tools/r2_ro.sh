python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CORTEX_LIB=variants/ro.so timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "prefill or cascade" 2>&1 | tail -1
for r in 1 2; do
for lib in "" variants/ro.so; do
  CORTEX_LIB=$lib timeout 200 python benchmarks/attn_step.py --fmha-only
  CORTEX_LIB=$lib timeout 200 python benchmarks/attn_step.py --layer-only
done
done
