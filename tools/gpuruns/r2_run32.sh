# r2 run 32: ncu of the bench's new dominant kernel (TSMTTSM D 58, L-blocks) and of TSMTTSM D 49 (the minimum)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmttsm d 58x58" "tsmttsm d 49x49"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r32_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r32_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
