# r2 run 11: full TSMM D retune (every candidate family) on the gather-free instantiations
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
W=$(python -c "print(','.join(str(i) for i in range(9,64) if i % 8))")
timeout 3100 python tools/autotune.py --ops tsmm --dtypes d --widths $W --time-budget 3000 --out gpurun_out/r11_tune_tsmm_d.json > gpurun_out/r11_tune_tsmm_d.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r11_tune_tsmm_d.json --dry | tail -60
