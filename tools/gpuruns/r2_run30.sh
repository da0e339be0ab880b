# r2 run 30: final validation of the run-29 merges -- smoke, GPU suite, bench (+ report), launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r30_smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/r30_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r30_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r30_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r30_bench_report.json > gpurun_out/r30_bench.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/r30_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r30_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sub > gpurun_out/r30_launches_bench.log 2>&1; echo launches rc=$?
