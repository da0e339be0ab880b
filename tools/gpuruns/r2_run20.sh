# r2 run 20: validate the run-19 merges (smoke, GPU suite, bench), then a heated retune of the
# FP64-bound D widths (TSMTTSM 25-64, TSMM 33-64 where the sweep is below 90 %)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r20_smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r20_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r20_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r20_bench_report.json > gpurun_out/r20_bench.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/r20_bench.log
W1=33,34,35,36,37,38,39,40,41,42,43,44,45,46,47,48,49,50,51,52,53,54,55,57,58,59,60,61,62,63
timeout 2400 python tools/autotune.py --ops tsmttsm --dtypes d --widths $W1 --heat 4 --reps 3 --time-budget 2300 --out gpurun_out/r20_tune_tsmttsm_d.json > gpurun_out/r20_tune_tsmttsm_d.log 2>&1; echo tune tsmttsm rc=$?
python tools/merge_tune.py gpurun_out/r20_tune_tsmttsm_d.json --dry
