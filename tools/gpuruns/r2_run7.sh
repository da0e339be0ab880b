# r2 run 7: L-blocks (TSMTTSM D) validation and tuning; reverted edge code check
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "lblocks or win16 or cstb_edge or inline_edge or every_family" > gpurun_out/r7_pytest.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r7_pytest.log
W=$(python -c "print(','.join(str(i) for i in range(9,64) if 1 <= i % 8 <= 6))")
timeout 1500 python tools/autotune.py --ops tsmttsm --dtypes d --widths $W --filter "c.get('LB')" --time-budget 1400 --out gpurun_out/r7_tune_lb.json > gpurun_out/r7_tune_lb.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r7_tune_lb.json --dry | tail -50
