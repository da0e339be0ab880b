timeout 1200 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x > gpurun_out/pytest_kern14.log 2>&1; echo kern rc=$?; tail -n 5 gpurun_out/pytest_kern14.log
cp tune/b200.json tune/b200_prev.json
timeout 3000 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d,z --widths 8-64 --time-budget 2600 > gpurun_out/autotune14.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r14.json
tail -n 2 gpurun_out/autotune14.log
