# r20: parity of multi-edge / complex-as-real / partial-tile dispatch; retune; bench + sweep
timeout 1200 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu20.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu20.log
timeout 2400 python tools/autotune.py --ops tsmttsm --dtypes d,z --widths 9-64 --filter "c.get('impl', 0) >= 1" --keep-better --time-budget 2100 > gpurun_out/autotune20a.log 2>&1; echo rc=$?
timeout 1500 python tools/autotune.py --ops tsmm --dtypes z,d --widths 9-64 --filter "c.get('impl', 0) == 3" --keep-better --time-budget 1200 > gpurun_out/autotune20b.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r20.json
