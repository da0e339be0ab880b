# r2 run 27: heated retune of the odd FP64-bound TSMM D widths over the new 12/16-warp kernel-1 candidates
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python tools/autotune.py --ops tsmm --dtypes d --widths 37,39,41,43,45,47,49,50,51,53,54,55,57,58,59,61,62,63 --heat 4 --reps 3 --filter "c.get('impl') in (1, 2) and c['NT'] >= 416" --time-budget 1700 --out gpurun_out/r27_tune_tsmm_d.json > gpurun_out/r27_tune_tsmm_d.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r27_tune_tsmm_d.json --dry
