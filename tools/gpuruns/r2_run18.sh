# r2 run 18: solo-finisher grid reduction (parity), small-K in the paper's metric with write vs clean L2 flush,
# in-sweep vs isolated timing of the HBM-bound TSMTTSM widths that lose in the sweep, ncu of D 16 / 24 / 42
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/r18_pytest_parity.log 2>&1; echo pytest rc=$?; tail -n 2 gpurun_out/r18_pytest_parity.log
for fl in write read; do
  timeout 600 python tools/smallk.py --widths 4,8,32,64 --Ks 1e5,3e5,1e6,3e6,1e7 --flush $fl --json gpurun_out/r18_smallk_$fl.json > gpurun_out/r18_smallk_$fl.log 2>&1; echo smallk $fl rc=$?
done
for w in 1 2 3 8 9 16 24 13; do
  timeout 300 python tools/order_probe.py --dtype d --light tsmttsm:$w --heavy tsmttsm:$((w-1>0?w-1:1)) --reps 15 >> gpurun_out/r18_order.log 2>&1; echo order $w rc=$?
done
cat gpurun_out/r18_order.log
NCU="ncu --set full --clock-control none --import-source on -s 2 -c 1"
for spec in "tsmttsm d 16x16" "tsmttsm d 24x24" "tsmttsm d 42x42"; do
  set -- $spec
  timeout 400 $NCU -k regex:$1 -o gpurun_out/r18_ncu_$1_$2_$3 python tools/quick_time.py --ops $1 --dtypes $2 --shapes $3 --reps 1 > gpurun_out/r18_ncu_$1_$2_$3.log 2>&1; echo "ncu $spec rc=$?"
done
