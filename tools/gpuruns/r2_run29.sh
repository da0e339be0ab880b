# r2 run 29: the 12/16-warp kernel-1 candidates at the remaining FP64-bound TSMM D widths
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python tools/autotune.py --ops tsmm --dtypes d --widths 33,35,42,44,46,47,48,49,52,56,57,58,60,64 --heat 4 --reps 3 --filter "c.get('impl') in (1, 2) and c['NT'] >= 416" --time-budget 1100 --out gpurun_out/r29_tune_tsmm_d.json > gpurun_out/r29_tune_tsmm_d.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r29_tune_tsmm_d.json --dry
