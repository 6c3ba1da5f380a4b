mkdir -p gpurun_out
timeout 600 python tools/diag_8b.py > gpurun_out/diag_8b.log 2>&1; echo rc $?
timeout 600 python tools/diag_8b.py --knob FMHA_PLO=0 > gpurun_out/diag_8b_plo.log 2>&1; echo rc $?
CORTEX_TC_ATTN=0 timeout 600 python tools/diag_8b.py > gpurun_out/diag_8b_mma.log 2>&1; echo rc $?
cat gpurun_out/diag_8b.log; echo ---; cat gpurun_out/diag_8b_plo.log; echo ---; cat gpurun_out/diag_8b_mma.log
