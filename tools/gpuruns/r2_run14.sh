# r2 run 14: the Z 21 complex-as-real L-block launch failure; ncu of the headline's dominant kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/repro_launch.py tsmttsm z 21 21 '{"AP": 42, "BP": 42, "LB": 1, "MT": 3, "NT": 96, "NTL": 5, "R": 16, "ZR": 1, "ctas": 4, "impl": 1, "stages": 4}' 2>&1 | tail -20
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmm d 63x63" "tsmttsm d 63x63" "tsmm d 57x57"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r14_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r14_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
