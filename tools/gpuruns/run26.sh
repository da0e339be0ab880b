# r26: validate edge v2 / SMSP spreading, then a fresh full retune on the final kernel source
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_next_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu26.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu26.log
timeout 4200 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d,z --widths 1-64 --time-budget 3900 > gpurun_out/autotune26.log 2>&1; echo autotune rc=$?
timeout 900 python tools/autotune.py --ops tsmttsm,tsmm --dtypes d,z --shapes 1x64,64x1,16x48,48x16,1x2,2x1,3x5,5x3,7x2,13x29,29x13,33x17,17x33,5x64,64x5,1x7,9x1,63x64,64x63 --time-budget 800 > gpurun_out/autotune26n.log 2>&1; echo autotune-n rc=$?
cp tune/b200.json gpurun_out/b200_r26.json
