for s in "qkv 768" "gate_up 512" "down 512" "o 768"; do
  set -- $s
  CORTEX_LIB=variants/libcortex_gtrace.so timeout 120 python benchmarks/gemm_trace.py $1 $2 0 2>&1 | grep -v "^exit" | tail -8
done
