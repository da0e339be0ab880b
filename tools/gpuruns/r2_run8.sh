# r2 run 8: full GPU test suite on the current code + smoke + bench + order probe
bash tools/gpuruns/ab_old_new.sh 2>&1 | tee gpurun_out/r8_ab.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8_smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/r8_smoke.log
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r8_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 6 gpurun_out/r8_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r8_bench_report.json > gpurun_out/r8_bench.log 2>&1; echo bench rc=$?; tail -c 600 gpurun_out/r8_bench.log
for spec in "z tsmttsm:1 tsmm:64" "d tsmttsm:1 tsmm:64" "d tsmttsm:8 tsmm:57"; do set -- $spec; timeout 120 python tools/order_probe.py --dtype $1 --light $2 --heavy $3; done
