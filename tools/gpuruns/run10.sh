timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu10.log 2>&1; echo pytest rc=$?; tail -n 15 gpurun_out/pytest_gpu10.log
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths 16,24,32,40,48,49,56,64 --reps 5 > gpurun_out/qt10.log 2>&1; echo qt rc=$?
