mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for kn in DECODE_PERSIST=0 DECODE_PERSIST=1; do
  CORTEX_KNOBS=$kn timeout 300 python benchmarks/attn_step.py --private-only
done
CORTEX_LIB=variants/decstatic.so CORTEX_KNOBS=DECODE_PERSIST=1 timeout 300 python benchmarks/attn_step.py --private-only
CORTEX_KNOBS=DECODE_PERSIST=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_decode -c 2 -o gpurun_out/r2u_ncu_persist python benchmarks/attn_step.py --private-only > gpurun_out/r2u_ncu1.log 2>&1; echo ncu $?
CORTEX_KNOBS=DECODE_PERSIST=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_decode -c 2 -o gpurun_out/r2u_ncu_item python benchmarks/attn_step.py --private-only > gpurun_out/r2u_ncu2.log 2>&1; echo ncu $?
