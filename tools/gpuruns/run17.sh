timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu17.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu17.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report17.json > gpurun_out/bench17.log 2>&1; echo bench rc=$?; tail -c 600 gpurun_out/bench17.log
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths $W --reps 3 --json gpurun_out/sweep17_square.json > gpurun_out/sweep17_square.log 2>&1; echo sq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48 --K 33554432 --reps 3 --json gpurun_out/sweep17_nonsq.json > gpurun_out/sweep17_nonsq.log 2>&1; echo nonsq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d --shapes 8x8 --K 1000000 --reps 10 --json gpurun_out/sweep17_cfg0.json > gpurun_out/sweep17_cfg0.log 2>&1; echo cfg0 rc=$?
