timeout 1200 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x > gpurun_out/pytest_kern13.log 2>&1; echo kern rc=$?; tail -n 5 gpurun_out/pytest_kern13.log
bash tools/ncu_run.sh r01b tsmttsm d 48x48 64x64
bash tools/ncu_run.sh r01b tsmttsm z 33x33 48x48
bash tools/ncu_run.sh r01b tsmm d 64x64 41x41
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r01b_launches_bench.log 2>&1; echo launches rc=$?
