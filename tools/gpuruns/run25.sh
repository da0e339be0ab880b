# r25: tune pair+edge / remaining candidates for the padding widths; full tests on the final source; bench; sweeps; ncu
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "edge_warp or pair" > gpurun_out/pytest_gpu25a.log 2>&1; echo pytest-a rc=$?; tail -n 2 gpurun_out/pytest_gpu25a.log
timeout 1500 python tools/autotune.py --ops tsmttsm --dtypes d --widths 33,34,35,41,42,43,49,50,51,57,58,59 --keep-better --time-budget 1300 > gpurun_out/autotune25.log 2>&1; echo autotune rc=$?
timeout 1500 python tools/autotune.py --ops tsmttsm --dtypes z --widths 17-39 --filter "c.get('ZR') and c.get('EDGE')" --keep-better --time-budget 1300 > gpurun_out/autotune25z.log 2>&1; echo autotune-z rc=$?
cp tune/b200.json gpurun_out/b200_r25.json
python tools/gen_instances.py > /dev/null && python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build25.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu25.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu25.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report25.json > gpurun_out/bench25.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/bench25.log
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --widths $W --reps 3 --json gpurun_out/sweep25_square.json > gpurun_out/sweep25_square.log 2>&1; echo sq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48 --K 33554432 --reps 3 --json gpurun_out/sweep25_nonsq.json > gpurun_out/sweep25_nonsq.log 2>&1; echo nonsq rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm --dtypes d --shapes 8x8 --K 1000000 --reps 10 --json gpurun_out/sweep25_cfg0.json > gpurun_out/sweep25_cfg0.log 2>&1; echo cfg0 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches25.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/launches25_bench.log 2>&1; echo launches rc=$?
