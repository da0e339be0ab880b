# r28: fresh-container re-check -- GPU tests, smoke, bench, sweeps, launch list, dram traffic, ncu of weak widths
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke28.log 2>&1; echo smoke rc=$?; tail -n 3 gpurun_out/smoke28.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report28.json > gpurun_out/bench28.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/bench28.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu28.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu28.log
timeout 600 python bench.py --steps 2 --warmup 3 --force-comm --no-e2e --no-cpu > gpurun_out/bench28_comm.log 2>&1; echo bench-comm rc=$?; tail -c 200 gpurun_out/bench28_comm.log
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths $W --reps 3 --json gpurun_out/sweep28_square.json > gpurun_out/sweep28_square.log 2>&1; echo sq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48 --K 33554432 --reps 3 --json gpurun_out/sweep28_nonsq.json > gpurun_out/sweep28_nonsq.log 2>&1; echo nonsq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d --shapes 8x8 --K 1000000 --reps 10 --json gpurun_out/sweep28_cfg0.json > gpurun_out/sweep28_cfg0.log 2>&1; echo cfg0 rc=$?
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths 8,32,64 --Ks 10000,100000,1000000,10000000,100000000 --reps 5 --json gpurun_out/smallk28.json > gpurun_out/smallk28.log 2>&1; echo smallk rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches28.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/launches28_bench.log 2>&1; echo launches rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tsm -o gpurun_out/traffic28 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 1 > gpurun_out/traffic28.log 2>&1; echo traffic rc=$?
bash tools/ncu_run.sh r28 tsmttsm d 56x56 50x50
bash tools/ncu_run.sh r28 tsmm d 63x63
