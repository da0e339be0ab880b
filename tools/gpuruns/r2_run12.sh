# r2 run 12: Z retune of the run-9 merges, then the evidence pass on the final tables:
# smoke, full GPU suite, bench (+ table), ncu launch list of the bench, dram traffic per kernel
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python tools/autotune.py --ops tsmttsm --dtypes z --widths 9,17,21,26,33,37,53 --time-budget 800 --out gpurun_out/r12_tune_z.json > gpurun_out/r12_tune_z.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r12_tune_z.json --dry | tail -10
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r12_smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/r12_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r12_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 4 gpurun_out/r12_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r12_bench_report.json > gpurun_out/r12_bench.log 2>&1; echo bench rc=$?; tail -c 400 gpurun_out/r12_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r12_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sub > gpurun_out/r12_launches_bench.log 2>&1; echo launches rc=$?
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tsm -o gpurun_out/r12_traffic python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 1 > gpurun_out/r12_traffic.log 2>&1; echo traffic rc=$?
