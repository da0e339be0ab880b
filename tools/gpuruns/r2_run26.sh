# r2 run 26: validation of the run-25 merges (smoke, GPU suite, bench) and a last heated Z retune
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r26_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r26_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r26_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r26_bench_report.json > gpurun_out/r26_bench.log 2>&1; echo bench rc=$?; tail -c 200 gpurun_out/r26_bench.log
timeout 1500 python tools/autotune.py --ops tsmm --dtypes z --widths 57,61,64 --heat 2 --reps 3 --time-budget 600 --out gpurun_out/r26_tune_tsmm_z.json > gpurun_out/r26_tune_tsmm_z.log 2>&1; echo tune tsmm z rc=$?
python tools/merge_tune.py gpurun_out/r26_tune_tsmm_z.json --dry
timeout 1800 python tools/autotune.py --ops tsmttsm --dtypes z --widths 19,20,23,24,28,32,39,44,45,46,47,48,51,52,55,56,59,60,61,62,63,64 --heat 2 --reps 3 --time-budget 1700 --out gpurun_out/r26_tune_tsmttsm_z.json > gpurun_out/r26_tune_tsmttsm_z.log 2>&1; echo tune tsmttsm z rc=$?
python tools/merge_tune.py gpurun_out/r26_tune_tsmttsm_z.json --dry
