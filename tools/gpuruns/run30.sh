# r30: FP64-pipe concurrency probe; 3M defaults merged (r29) -- parity; Z sweep; D/Z warp-order A/B; D compute-width retune (both orders)
./tools/probes/fp64_mix > gpurun_out/fp64_mix30.log 2>&1; echo probe rc=$?; cat gpurun_out/fp64_mix30.log
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu30.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu30.log
W=$(python -c "print(','.join(str(i) for i in range(17,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes z --widths $W --reps 3 --json gpurun_out/sweep30_z.json > gpurun_out/sweep30_z.log 2>&1; echo zsweep rc=$?
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes z --widths $W --reps 3 --toggle-order --json gpurun_out/sweep30_z_tog.json > gpurun_out/sweep30_z_tog.log 2>&1; echo ztog rc=$?
W=$(python -c "print(','.join(str(i) for i in range(33,65)))")
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 3 --json gpurun_out/sweep30_d.json > gpurun_out/sweep30_d.log 2>&1; echo dsweep rc=$?
timeout 900 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --widths $W --reps 3 --toggle-order --json gpurun_out/sweep30_d_tog.json > gpurun_out/sweep30_d_tog.log 2>&1; echo dtog rc=$?
timeout 600 python tools/quick_time.py --ops tsmttsm,tsmm --dtypes z --shapes 1x64,64x1,16x48 --K 33554432 --reps 3 --json gpurun_out/sweep30_nonsq.json > gpurun_out/sweep30_nonsq.log 2>&1; echo nonsq rc=$?
cp tune/b200.json gpurun_out/b200_r30.json
timeout 3000 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d --widths 33-64 --time-budget 2700 --out gpurun_out/b200_r30.json > gpurun_out/autotune30.log 2>&1; echo autotune rc=$?
