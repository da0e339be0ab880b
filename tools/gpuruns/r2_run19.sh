# r2 run 19: re-tune the HBM-bound widths that lose 6-15 % in the bench sweep, under the sweep's
# power-capped clock (autotune --heat), then a dry merge
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python tools/autotune.py --ops tsmttsm --dtypes d --widths 1,2,3,4,5,6,8,9,10,13,15,16,17,20,24,28 --heat 4 --reps 5 --time-budget 1400 --out gpurun_out/r19_tune_tsmttsm_d.json > gpurun_out/r19_tune_tsmttsm_d.log 2>&1; echo tune d rc=$?
timeout 500 python tools/autotune.py --ops tsmttsm --dtypes z --widths 1,2,3 --heat 4 --reps 5 --time-budget 400 --out gpurun_out/r19_tune_tsmttsm_z.json > gpurun_out/r19_tune_tsmttsm_z.log 2>&1; echo tune z rc=$?
timeout 600 python tools/autotune.py --ops tsmm --dtypes d --widths 5,35,37,39 --heat 4 --reps 5 --time-budget 500 --out gpurun_out/r19_tune_tsmm_d.json > gpurun_out/r19_tune_tsmm_d.log 2>&1; echo tune tsmm rc=$?
for f in tsmttsm_d tsmttsm_z tsmm_d; do python tools/merge_tune.py gpurun_out/r19_tune_$f.json --dry; done
