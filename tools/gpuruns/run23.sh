# r23: NVRTC-first plans (precompiled kcache) -- full GPU tests, bench, sweeps, ncu of weak widths
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu23.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu23.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report23.json > gpurun_out/bench23.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/bench23.log
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths $W --reps 3 --json gpurun_out/sweep23_square.json > gpurun_out/sweep23_square.log 2>&1; echo sq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48 --K 33554432 --reps 3 --json gpurun_out/sweep23_nonsq.json > gpurun_out/sweep23_nonsq.log 2>&1; echo nonsq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d --shapes 8x8 --K 1000000 --reps 10 --json gpurun_out/sweep23_cfg0.json > gpurun_out/sweep23_cfg0.log 2>&1; echo cfg0 rc=$?
bash tools/ncu_run.sh r23 tsmttsm d 56x56 50x50
bash tools/ncu_run.sh r23 tsmm d 63x63 50x50
