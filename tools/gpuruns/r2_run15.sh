# r2 run 15: validate native complex L-blocks; tune Z TSMTTSM with them (widths with an L-block gain)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "z_lblocks or zr_lblocks or lblocks" > gpurun_out/r15_pytest.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/r15_pytest.log
W=$(python -c "print(','.join(str(i) for i in range(9,64) if 1 <= i % 8 <= 6))")
timeout 2400 python tools/autotune.py --ops tsmttsm --dtypes z --widths $W --filter "c.get('LB')" --time-budget 2300 --out gpurun_out/r15_tune_z_lb.json > gpurun_out/r15_tune_z_lb.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r15_tune_z_lb.json --dry | tail -50
