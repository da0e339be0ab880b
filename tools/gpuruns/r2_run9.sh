# r2 run 9: evidence on the current kernels -- ncu launch list of the bench
# command, dram traffic per kernel over the D sweep, ncu --set full of the
# heaviest kernels, sanitizers (synccheck over the barrier / window / L-block
# families; memcheck and racecheck over all families)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
W=$(python -c "print(','.join(str(i) for i in range(1,65)))")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r9_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sub > gpurun_out/r9_launches_bench.log 2>&1; echo launches rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tsm -o gpurun_out/r9_traffic python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 1 > gpurun_out/r9_traffic.log 2>&1; echo traffic rc=$?
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmm d 63x63" "tsmttsm d 57x57" "tsmttsm d 64x64" "tsmm d 62x62" "tsmttsm d 49x49"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r9_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r9_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py --match cstb,l-blocks,dmma > gpurun_out/r9_san_synccheck.log 2>&1; echo synccheck rc=$?; tail -3 gpurun_out/r9_san_synccheck.log
