# r2 run 10: full TSMTTSM D retune (every candidate family) on the gather-free instantiations
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/gpuruns/ab_old_new.sh 2>&1 | head -6 | tee gpurun_out/r10_ab.log
W=$(python -c "print(','.join(str(i) for i in range(9,64) if i % 8))")
timeout 3100 python tools/autotune.py --ops tsmttsm --dtypes d --widths $W --time-budget 3000 --out gpurun_out/r10_tune_tsmttsm_d.json > gpurun_out/r10_tune_tsmttsm_d.log 2>&1; echo tune rc=$?
python tools/merge_tune.py gpurun_out/r10_tune_tsmttsm_d.json --dry | tail -60
