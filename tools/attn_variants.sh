for v in "" variants/libcortex_t32.so variants/libcortex_t64.so; do
  echo "== $v"; CORTEX_LIB=${v:-paper_2510_14126_b200/libcortex_b200.so} timeout -k 5 120 python benchmarks/attn_step.py 2>&1 | tail -1 | cut -c1-300
done
