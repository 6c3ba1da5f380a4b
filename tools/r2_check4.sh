set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1; echo build $?
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "argmax" > gpurun_out/r2d_pytest.log 2>&1; echo pytest $?
tail -5 gpurun_out/r2d_pytest.log
timeout 900 python tools/diag_8b_e2e.py > gpurun_out/r2d_diag_e2e.log 2>&1; echo diag $?
cat gpurun_out/r2d_diag_e2e.log | tail -25
