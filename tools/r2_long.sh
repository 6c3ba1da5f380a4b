mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python bench.py --gpus 1 --steps 1000 --warmup 5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2l_c2_1000.log 2>&1; echo c2 $?
timeout 2000 python bench.py --gpus 1 --steps 1500 --warmup 5 --workload config4 --no-cpu-baseline --no-shared-arm > gpurun_out/r2l_c4.log 2>&1; echo c4 $?
timeout 1200 python bench.py --gpus 1 --steps 300 --warmup 5 --workload config5 --no-cpu-baseline --no-shared-arm > gpurun_out/r2l_c5.log 2>&1; echo c5 $?
