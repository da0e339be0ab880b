timeout 600 python tools/quick_time.py --dtypes d,z --widths 1,2,4,8,16,24,32,40,48,56,64 --reps 5 > gpurun_out/qt2.log 2>&1; echo qt rc=$?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu2.log 2>&1; echo pytest rc=$?
tail -n 3 gpurun_out/pytest_gpu2.log
