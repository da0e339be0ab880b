timeout 3000 python tools/autotune.py --ops tsmm,tsmttsm --dtypes d,z --widths 1-64 --time-budget 2700 > gpurun_out/autotune11.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r11.json
timeout 300 python -m pytest tests/test_comm_gpu.py -m gpu -q > gpurun_out/pytest_comm11.log 2>&1; echo comm rc=$?; tail -n 3 gpurun_out/pytest_comm11.log
tail -n 3 gpurun_out/autotune11.log
