timeout 900 python -m pytest tests -m gpu -q -x -k "tsmttsm or int_mode or config1 or jit or explicit or walsh or nan or determinism" > gpurun_out/pytest_gpu6.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu6.log
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d,z --widths 1,2,4,8,12,16,20,24,32,40,48,56,64 --reps 5 > gpurun_out/qt6.log 2>&1; echo qt rc=$?
