# r22: parity of impl 4 / TSMM edge columns / strided views / N1 N2; retune TSMM kernels 3-4 and narrow TSMTTSM; small-K study
timeout 1800 python -m pytest tests/test_next_gpu.py tests/test_kernels_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu22.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu22.log
timeout 2400 python tools/autotune.py --ops tsmm --dtypes d,z --widths 8-64 --filter "c.get('impl', 0) in (3, 4)" --keep-better --time-budget 2100 > gpurun_out/autotune22a.log 2>&1; echo autotune-a rc=$?
timeout 900 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d,z --widths 1-8 --keep-better --time-budget 700 > gpurun_out/autotune22b.log 2>&1; echo autotune-b rc=$?
cp tune/b200.json gpurun_out/b200_r22.json
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths 8,32,64 --Ks 10000,100000,1000000,10000000,100000000 --reps 5 --json gpurun_out/smallk22.json > gpurun_out/smallk22.log 2>&1; echo smallk rc=$?
