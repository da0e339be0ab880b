# r2 run 5: validate the edge-DFMA restructuring (kernel family tests), then
# retune the edge variants (TSMM edge columns, TSMTTSM inline edge / edge warps)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_next_gpu.py -q -x > gpurun_out/r5_pytest.log 2>&1; echo pytest rc=$?; tail -n 4 gpurun_out/r5_pytest.log
W=$(python -c "print(','.join(str(i) for i in range(9,64) if i % 8))")
timeout 900 python tools/autotune.py --ops tsmm --dtypes d --widths $W --filter "c.get('EDGE')" --time-budget 840 --out gpurun_out/r5_tune_tsmm_d_edge.json > gpurun_out/r5_tune_tsmm_d_edge.log 2>&1; echo t1 rc=$?
timeout 900 python tools/autotune.py --ops tsmttsm --dtypes d --widths $W --filter "c.get('EI') or c.get('EDGE')" --time-budget 840 --out gpurun_out/r5_tune_tsmttsm_d_edge.json > gpurun_out/r5_tune_tsmttsm_d_edge.log 2>&1; echo t2 rc=$?
timeout 700 python tools/autotune.py --ops tsmm,tsmttsm --dtypes z --widths $W --filter "c.get('EI') or c.get('EDGE')" --time-budget 640 --out gpurun_out/r5_tune_z_edge.json > gpurun_out/r5_tune_z_edge.log 2>&1; echo t3 rc=$?
python tools/merge_tune.py gpurun_out/r5_tune_tsmm_d_edge.json --dry | tail -50
python tools/merge_tune.py gpurun_out/r5_tune_tsmttsm_d_edge.json --dry | tail -50
python tools/merge_tune.py gpurun_out/r5_tune_z_edge.json --dry | tail -80
