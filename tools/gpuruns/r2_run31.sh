# r2 run 31: the 12/16-warp kernel-1 candidates at the Z TSMM widths 17-32
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python tools/autotune.py --ops tsmm --dtypes z --widths 17,18,19,21,22,23,25,26,27,29,30,31,32 --heat 2 --reps 3 --filter "c.get('impl') in (1, 2) and c['NT'] >= 416" --time-budget 800 --out gpurun_out/r31_tune_tsmm_z.json > gpurun_out/r31_tune_tsmm_z.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r31_tune_tsmm_z.json --dry
