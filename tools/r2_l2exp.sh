for lib in gtrace gtrace_sameA gtrace_sameB gtrace_sameAB; do
  for s in "qkv 768" "down 512" "gate_up 512"; do
    set -- $s
    CORTEX_LIB=variants/libcortex_$lib.so timeout 120 python benchmarks/gemm_mainloop.py $1 $2 2>&1 | tail -1
  done
done
