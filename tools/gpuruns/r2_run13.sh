# r2 run 13: sanitizers over every family on the final kernels; ncu of the 3M Z kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/r13_san_$tool.log 2>&1
  echo $tool rc=$?; grep -h "SANITIZE_OK\|ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/r13_san_$tool.log
done
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmm z 64x64" "tsmm z 37x37" "tsmttsm z 57x57"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r13_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r13_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
