# r2 run 21: the 3M recomputed-sum variant (G3R) and the run-20 merges (kernel tests, full-size parity of the
# tuned plans, bench), then a heated retune of the FP64-bound TSMM D and 3M TSMM Z widths
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r21_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -m gpu -q > gpurun_out/r21_pytest.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r21_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/r21_bench_report.json > gpurun_out/r21_bench.log 2>&1; echo bench rc=$?; tail -c 200 gpurun_out/r21_bench.log
timeout 1700 python tools/autotune.py --ops tsmm --dtypes d --widths 41,42,43,45,46,47,49,50,51,53,54,55,57,58,59,61,62,63 --heat 4 --reps 3 --time-budget 1600 --out gpurun_out/r21_tune_tsmm_d.json > gpurun_out/r21_tune_tsmm_d.log 2>&1; echo tune d rc=$?
python tools/merge_tune.py gpurun_out/r21_tune_tsmm_d.json --dry
timeout 1300 python tools/autotune.py --ops tsmm --dtypes z --widths 29,30,33,37,41,45,49,50,57,61,64 --heat 2 --reps 3 --time-budget 1200 --out gpurun_out/r21_tune_tsmm_z.json > gpurun_out/r21_tune_tsmm_z.log 2>&1; echo tune z rc=$?
python tools/merge_tune.py gpurun_out/r21_tune_tsmm_z.json --dry
