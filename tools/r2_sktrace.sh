set -x
for s in "qkv 204 3" "o 204 4" "down 204 4" "qkv 204 2" "down 204 3"; do
  set -- $s
  CORTEX_LIB=variants/libcortex_sktrace.so timeout 120 python benchmarks/gemm_sk_trace.py $1 $2 $3
done
