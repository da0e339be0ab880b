# r32: measurement on the r30/r31-merged table -- GPU tests, smoke, bench, sweeps, launch list, dram traffic, ncu of the bench's top kernels and a 3M kernel
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke32.log 2>&1; echo smoke rc=$?; tail -n 3 gpurun_out/smoke32.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report32.json > gpurun_out/bench32.log 2>&1; echo bench rc=$?; tail -c 400 gpurun_out/bench32.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu32.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu32.log
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths $W --reps 3 --json gpurun_out/sweep32_square.json > gpurun_out/sweep32_square.log 2>&1; echo sq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48,48x16 --K 33554432 --reps 3 --json gpurun_out/sweep32_nonsq.json > gpurun_out/sweep32_nonsq.log 2>&1; echo nonsq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d --shapes 8x8 --K 1000000 --reps 10 --json gpurun_out/sweep32_cfg0.json > gpurun_out/sweep32_cfg0.log 2>&1; echo cfg0 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches32.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/launches32_bench.log 2>&1; echo launches rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tsm -o gpurun_out/traffic32 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 1 > gpurun_out/traffic32.log 2>&1; echo traffic rc=$?
bash tools/ncu_run.sh r32 tsmm d 63x63 57x57
bash tools/ncu_run.sh r32 tsmttsm d 50x50 64x64
bash tools/ncu_run.sh r32 tsmttsm z 32x32
