timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k edge > gpurun_out/pytest_edge15.log 2>&1; echo edge rc=$?; tail -n 4 gpurun_out/pytest_edge15.log
timeout 1800 python tools/autotune.py --ops tsmttsm --dtypes d,z --widths 9,10,11,17,18,19,25,26,27,33,34,35,41,42,43,49,50,51,57,58,59 --time-budget 1500 > gpurun_out/autotune15.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r15.json
