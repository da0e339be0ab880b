# r21: TMA-reduce probe, N1/N2 + edge parity, retune TSMTTSM, rebuild, full tests, bench, sweep, ncu
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_tmared tools/probes/tma_reduce_f64.cu -lcuda && timeout 60 /tmp/probe_tmared > gpurun_out/probe_tmared21.txt 2>&1; cat gpurun_out/probe_tmared21.txt
timeout 1500 python -m pytest tests/test_next_gpu.py tests/test_kernels_gpu.py tests/test_comm_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu21a.log 2>&1; echo pytest-a rc=$?; tail -n 3 gpurun_out/pytest_gpu21a.log
timeout 2700 python tools/autotune.py --ops tsmttsm --dtypes d,z --widths 9-64 --filter "c.get('impl', 0) >= 1" --keep-better --time-budget 2400 > gpurun_out/autotune21.log 2>&1; echo autotune rc=$?
cp tune/b200.json gpurun_out/b200_r21.json
python tools/gen_instances.py > /dev/null && python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build21.log 2>&1; echo build rc=$?
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu21.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu21.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report21.json > gpurun_out/bench21.log 2>&1; echo bench rc=$?; tail -c 400 gpurun_out/bench21.log
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths $W --reps 3 --json gpurun_out/sweep21_square.json > gpurun_out/sweep21_square.log 2>&1; echo sq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48 --K 33554432 --reps 3 --json gpurun_out/sweep21_nonsq.json > gpurun_out/sweep21_nonsq.log 2>&1; echo nonsq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d --shapes 8x8 --K 1000000 --reps 10 --json gpurun_out/sweep21_cfg0.json > gpurun_out/sweep21_cfg0.log 2>&1; echo cfg0 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches21.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/launches21_bench.log 2>&1; echo launches rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tsm -o gpurun_out/traffic21 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 1 > gpurun_out/traffic21.log 2>&1; echo traffic rc=$?
