timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "family or edge or cstationary or square or int_mode" > gpurun_out/pytest_gpu18.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu18.log
timeout 3000 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d,z --widths 8-64 --time-budget 2700 > gpurun_out/autotune18.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r18.json
