set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python tools/quick_time.py --dtypes d --widths 1,8,16,32,48,64 --reps 5 > gpurun_out/qt1.log 2>&1; echo qt rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu1.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/smoke.log gpurun_out/qt1.log gpurun_out/pytest_gpu1.log
