# r2 run 25: heated retune of the FP64-bound shapes not yet re-picked at the sweep's clock
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python tools/autotune.py --ops tsmttsm --dtypes d --widths 44,45,46,47,48,52,53,54,55,56,64 --heat 4 --reps 3 --time-budget 1400 --out gpurun_out/r25_tune_tsmttsm_d.json > gpurun_out/r25_tune_tsmttsm_d.log 2>&1; echo tune tsmttsm d rc=$?
python tools/merge_tune.py gpurun_out/r25_tune_tsmttsm_d.json --dry
timeout 900 python tools/autotune.py --ops tsmm --dtypes d --widths 44,48,52,56,60,64 --heat 4 --reps 3 --time-budget 800 --out gpurun_out/r25_tune_tsmm_d.json > gpurun_out/r25_tune_tsmm_d.log 2>&1; echo tune tsmm d rc=$?
python tools/merge_tune.py gpurun_out/r25_tune_tsmm_d.json --dry
timeout 1500 python tools/autotune.py --ops tsmm --dtypes z --widths 36,38,39,40,42,43,44,46,47,48,51,52,53,54,55,56,58,59,60,62,63 --heat 2 --reps 3 --time-budget 1400 --out gpurun_out/r25_tune_tsmm_z.json > gpurun_out/r25_tune_tsmm_z.log 2>&1; echo tune tsmm z rc=$?
python tools/merge_tune.py gpurun_out/r25_tune_tsmm_z.json --dry
