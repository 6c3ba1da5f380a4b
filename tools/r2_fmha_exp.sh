mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
: > gpurun_out/r2z_fmha.jsonl
for lib in "" variants/fnosm.so variants/fnomma.so variants/fnone.so; do
  for kn in FMHA_2Q=-1 FMHA_2Q=0 FMHA_2Q=1 FMHA_PLO=0; do
    CORTEX_LIB=$lib CORTEX_KNOBS=$kn timeout 120 python benchmarks/attn_step.py --fmha-only > gpurun_out/r2z_one.log 2>&1
    echo "$lib $kn rc=$?" >> gpurun_out/r2z_fmha.jsonl
    grep '^{' gpurun_out/r2z_one.log >> gpurun_out/r2z_fmha.jsonl
  done
done
cat gpurun_out/r2z_fmha.jsonl
