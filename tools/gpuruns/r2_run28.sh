# r2 run 28: final evidence pass on the run-25..27 tables -- smoke, GPU suite, bench (+ report), reference arm,
# ncu launch list of the bench, ncu --set full of the dominant kernel (new 12-warp TSMM D 63) and of TSMM D 55
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r28_smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/r28_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r28_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r28_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r28_bench_report.json > gpurun_out/r28_bench.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/r28_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r28_bench_ref.log 2>&1; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r28_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sub > gpurun_out/r28_launches_bench.log 2>&1; echo launches rc=$?
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmm d 63x63" "tsmm d 55x55"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r28_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r28_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
