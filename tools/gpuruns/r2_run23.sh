# r2 run 23: evidence pass on the run-19..22 tables and the G3R kernels -- smoke, GPU suite, bench (+ report),
# reference arm, ncu launch list of the bench, ncu of the dominant kernels, order probe after the TSMM sweep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r23_smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/r23_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r23_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r23_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r23_bench_report.json > gpurun_out/r23_bench.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/r23_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r23_bench_ref.log 2>&1; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r23_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sub > gpurun_out/r23_launches_bench.log 2>&1; echo launches rc=$?
for w in 1 2 4; do timeout 300 python tools/order_probe.py --dtype d --light tsmttsm:$w --heavy tsmm:64 --reps 15 >> gpurun_out/r23_order.log 2>&1; done; cat gpurun_out/r23_order.log
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmm d 63x63" "tsmttsm d 63x63" "tsmm z 64x64"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r23_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r23_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
