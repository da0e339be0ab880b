# r41: parity of the restored TSMM D 63 default, Z bench line (3M kernels), D bench again
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "square or full_size" > gpurun_out/pytest_gpu41.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu41.log
timeout 900 python bench.py --dtype z --steps 3 --warmup 3 --no-e2e --no-cpu --report gpurun_out/bench_report41_z.json > gpurun_out/bench41_z.log 2>&1; echo bench-z rc=$?; tail -c 300 gpurun_out/bench41_z.log
timeout 900 python bench.py --steps 5 --warmup 3 --report gpurun_out/bench_report41.json > gpurun_out/bench41.log 2>&1; echo bench rc=$?; tail -c 300 gpurun_out/bench41.log
