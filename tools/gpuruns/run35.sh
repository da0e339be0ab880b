# r35: fused peer reduction after the fence change -- tests + world-1 fixed costs; ncu of small-K launches (K = 10^4) to split the fixed cost
timeout 900 python -m pytest tests/test_peer_gpu.py -m gpu -q -x > gpurun_out/pytest_peer35.log 2>&1; echo pytest-peer rc=$?; tail -n 3 gpurun_out/pytest_peer35.log
timeout 900 python tools/peer_time.py --dtypes d --Ks 10000,100000,1000000 --json gpurun_out/peer_time35.json > gpurun_out/peer_time35.log 2>&1; echo peer-time rc=$?; tail -n 9 gpurun_out/peer_time35.log
timeout 600 ncu --set full --clock-control none -k regex:tsm -s 3 -c 2 -o gpurun_out/r35_smallk python tools/quick_time.py --ops tsmttsm,tsmm --dtypes d --shapes 8x8 --K 10000 --reps 1 > gpurun_out/r35_smallk.log 2>&1; echo ncu-smallk rc=$?
