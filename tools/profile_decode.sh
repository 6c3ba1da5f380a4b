#!/bin/bash
# ncu --set full of the private-context decode kernels (per-split and flat) on the
# config-2 layer shape of benchmarks/attn_step.py
mkdir -p gpurun_out
timeout -k 5 120 python benchmarks/attn_step.py --once > /dev/null 2>&1 && echo plain-ok
CORTEX_FLAT_DECODE=0 timeout -k 5 600 ncu --set full --clock-control none --import-source on \
  -k regex:"paged_decode" -s 1 -c 1 -o gpurun_out/prof_dec_split$1 \
  python benchmarks/attn_step.py --once > gpurun_out/ncu_dec.log 2>&1; echo ncu $?
timeout -k 5 600 ncu --set full --clock-control none --import-source on \
  -k regex:"paged_decode" -s 1 -c 1 -o gpurun_out/prof_dec_flat$1 \
  python benchmarks/attn_step.py --once >> gpurun_out/ncu_dec.log 2>&1; echo ncu $?
