# r29: 3M (Gauss) Z kernels -- parity tests, then autotune Z widths 17..64 over the 3M candidates only (keep-better)
timeout 1200 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "3m" > gpurun_out/pytest_gpu29.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu29.log
cp tune/b200.json gpurun_out/b200_pre29.json
timeout 4200 python tools/autotune.py --ops tsmttsm,tsmm --dtypes z --widths 17-64 --filter "c.get('G3')" --keep-better --time-budget 3900 > gpurun_out/autotune29.log 2>&1; echo autotune rc=$?
timeout 600 python tools/autotune.py --ops tsmttsm,tsmm --dtypes z --shapes 16x48,48x16,64x1,1x64 --filter "c.get('G3')" --keep-better --time-budget 500 --K 33554432 > gpurun_out/autotune29n.log 2>&1; echo autotune-n rc=$?
cp tune/b200.json gpurun_out/b200_r29.json
