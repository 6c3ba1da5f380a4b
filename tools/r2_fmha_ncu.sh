mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -c 8 -o gpurun_out/r2s_ncu_fmha python benchmarks/attn_step.py --once > gpurun_out/r2s_ncu_fmha.log 2>&1; echo ncu $?
tail -3 gpurun_out/r2s_ncu_fmha.log
