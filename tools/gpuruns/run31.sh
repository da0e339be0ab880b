# r31: fresh full retune of the shapes r30 did not retune (Z 1..64 all candidate families incl. 3M and warp order, D 1..32, non-square) into a copy of the table
cp tune/b200.json gpurun_out/b200_r31.json
timeout 3600 python tools/autotune.py --ops tsmttsm,tsmm --dtypes z --widths 1-64 --time-budget 3300 --out gpurun_out/b200_r31.json > gpurun_out/autotune31z.log 2>&1; echo autotune-z rc=$?
timeout 1500 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d --widths 1-32 --time-budget 1300 --out gpurun_out/b200_r31.json > gpurun_out/autotune31d.log 2>&1; echo autotune-d rc=$?
timeout 900 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48,48x16 --K 33554432 --time-budget 800 --out gpurun_out/b200_r31.json > gpurun_out/autotune31n.log 2>&1; echo autotune-n rc=$?
W=$(python -c "print(','.join(str(i) for i in range(1,33)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 3 --json gpurun_out/sweep31_d.json > gpurun_out/sweep31_d.log 2>&1; echo dsweep rc=$?
W=$(python -c "print(','.join(str(i) for i in range(1,17)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes z --widths $W --reps 3 --json gpurun_out/sweep31_z.json > gpurun_out/sweep31_z.log 2>&1; echo zsweep rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48,48x16 --K 33554432 --reps 3 --json gpurun_out/sweep31_nonsq.json > gpurun_out/sweep31_nonsq.log 2>&1; echo nonsq rc=$?
