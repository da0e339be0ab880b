# r36: final validation on the final kernel source -- smoke, bench, full GPU tests, bench launch list
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke36.log 2>&1; echo smoke rc=$?; tail -n 3 gpurun_out/smoke36.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report36.json > gpurun_out/bench36.log 2>&1; echo bench rc=$?; tail -c 400 gpurun_out/bench36.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu36.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu36.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench36_ref.log 2>&1; echo ref rc=$?; tail -c 300 gpurun_out/bench36_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches36.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/launches36_bench.log 2>&1; echo launches rc=$?
