#!/bin/bash
# ncu --set full of the attention pieces of one config-2 layer (benchmarks/attn_step.py)
set -x
mkdir -p gpurun_out
timeout -k 5 120 python benchmarks/attn_step.py --once && echo plain-ok
timeout -k 5 600 ncu --set full --clock-control none --import-source on \
  -k regex:"paged_decode|decode_combine|fmha" -s 4 -c 4 -o gpurun_out/prof_attn_step${1:-} \
  python benchmarks/attn_step.py --once > gpurun_out/ncu_attn_step.log 2>&1; echo ncu $?
