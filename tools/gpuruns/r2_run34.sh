# r2 run 34: the final in-tree artifacts (rebuilt after the reverted experiment): smoke, parity suite, bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r34_smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/r34_smoke.log
timeout 900 python -m pytest tests/test_parity_gpu.py -q > gpurun_out/r34_pytest_parity.log 2>&1; echo pytest rc=$?; tail -n 2 gpurun_out/r34_pytest_parity.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r34_bench_report.json > gpurun_out/r34_bench.log 2>&1; echo bench rc=$?; tail -c 200 gpurun_out/r34_bench.log
