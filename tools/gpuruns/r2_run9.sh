# r2 run 9: complex-as-real L-blocks -- tests and tune (Z TSMTTSM), synccheck on the barrier / L-block families
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "zr_lblocks or lblocks" > gpurun_out/r9_pytest.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r9_pytest.log
W=$(python -c "print(','.join(str(i) for i in range(9,65) if 2 <= (2*i) % 8 <= 6))")
timeout 1700 python tools/autotune.py --ops tsmttsm --dtypes z --widths $W --filter "c.get('LB')" --time-budget 1600 --out gpurun_out/r9_tune_zr_lb.json > gpurun_out/r9_tune_zr_lb.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r9_tune_zr_lb.json --dry | tail -60
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py --match cstb,l-blocks > gpurun_out/r9_san_synccheck.log 2>&1; echo synccheck rc=$?; tail -3 gpurun_out/r9_san_synccheck.log
