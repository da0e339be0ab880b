# r43: final measurement on the final table -- smoke, bench, full GPU tests, sweeps, launch list, dram traffic, ncu
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke43.log 2>&1; echo smoke rc=$?; tail -n 3 gpurun_out/smoke43.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report43.json > gpurun_out/bench43.log 2>&1; echo bench rc=$?; tail -c 400 gpurun_out/bench43.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu43.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu43.log
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths $W --reps 3 --json gpurun_out/sweep43_square.json > gpurun_out/sweep43_square.log 2>&1; echo sq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48,48x16 --K 33554432 --reps 3 --json gpurun_out/sweep43_nonsq.json > gpurun_out/sweep43_nonsq.log 2>&1; echo nonsq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d --shapes 8x8 --K 1000000 --reps 10 --json gpurun_out/sweep43_cfg0.json > gpurun_out/sweep43_cfg0.log 2>&1; echo cfg0 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches43.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/launches43_bench.log 2>&1; echo launches rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tsm -o gpurun_out/traffic43 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 1 > gpurun_out/traffic43.log 2>&1; echo traffic rc=$?
bash tools/ncu_run.sh r43 tsmm d 63x63
bash tools/ncu_run.sh r43 tsmttsm d 34x34
bash tools/ncu_run.sh r43 tsmttsm z 17x17
