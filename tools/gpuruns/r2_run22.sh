# r2 run 22: ncu (source-correlated) of the 3M Z kernels after G3R; heated retune of the FP64-bound Z widths
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmm z 64x64" "tsmttsm z 57x57" "tsmm z 41x41"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r22_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r22_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
timeout 2700 python tools/autotune.py --ops tsmttsm --dtypes z --widths 17,18,21,22,25,26,27,29,30,31,33,34,35,36,37,38,40,41,42,43,49,50,53,54,57,58 --heat 2 --reps 3 --time-budget 2600 --out gpurun_out/r22_tune_tsmttsm_z.json > gpurun_out/r22_tune_tsmttsm_z.log 2>&1; echo tune tsmttsm z rc=$?
python tools/merge_tune.py gpurun_out/r22_tune_tsmttsm_z.json --dry
timeout 1000 python tools/autotune.py --ops tsmm --dtypes z --widths 21,25,29,30,31,32,33,34,35 --heat 2 --reps 3 --time-budget 900 --out gpurun_out/r22_tune_tsmm_z.json > gpurun_out/r22_tune_tsmm_z.log 2>&1; echo tune tsmm z rc=$?
python tools/merge_tune.py gpurun_out/r22_tune_tsmm_z.json --dry
