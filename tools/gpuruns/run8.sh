timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu8.log 2>&1; echo pytest rc=$?; tail -n 4 gpurun_out/pytest_gpu8.log
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths 1,2,4,8,12,16,24,32,33,40,48,56,64 --reps 5 > gpurun_out/qt8.log 2>&1; echo qt rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 --report gpurun_out/bench_report8.json > gpurun_out/bench8.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/bench8.log
