mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2n_launches_timed.csv python bench.py --gpus 1 --steps 3 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2n_ncu.log 2>&1; echo ncu $?
cp gpurun_out/ncu_window_algorithmic.json gpurun_out/r2n_ncu_window_algorithmic.json
CORTEX_NCU_TIMED=1 timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:fmha2 -c 2 -o gpurun_out/r2n_ncu_fmha2_step python bench.py --gpus 1 --steps 2 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2n_ncu_full.log 2>&1; echo ncufull $?
