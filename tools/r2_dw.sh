python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
for lib in "" variants/dw2.so; do
  CORTEX_LIB=$lib timeout 200 python benchmarks/attn_step.py --layer-only
done
done
