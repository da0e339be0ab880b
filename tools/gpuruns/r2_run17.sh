# r2 run 17: evidence pass on the final tables -- smoke, full GPU suite, bench (+ report), launch list, reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r17_smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/r17_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r17_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 4 gpurun_out/r17_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r17_bench_report.json > gpurun_out/r17_bench.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/r17_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r17_bench_ref.log 2>&1; echo ref rc=$?; tail -c 300 gpurun_out/r17_bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r17_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sub > gpurun_out/r17_launches_bench.log 2>&1; echo launches rc=$?
