# r40: final validation on the final table -- smoke, bench, full GPU tests, bench launch list, ncu of the bench's largest-share kernel
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke40.log 2>&1; echo smoke rc=$?; tail -n 3 gpurun_out/smoke40.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report40.json > gpurun_out/bench40.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/bench40.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu40.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu40.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches40.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/launches40_bench.log 2>&1; echo launches rc=$?
bash tools/ncu_run.sh r40 tsmm d 63x63 47x47
