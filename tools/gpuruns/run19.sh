# r19: parity of the pair / k-row-remap / rho variants, retune DMMA kernels, ncu of the top kernels
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu19.log 2>&1; echo pytest rc=$?; tail -n 3 gpurun_out/pytest_gpu19.log
timeout 1800 python tools/autotune.py --ops tsmttsm --dtypes d,z --widths 8-64 --filter "c.get('impl', 0) >= 1" --keep-better --time-budget 1500 > gpurun_out/autotune19a.log 2>&1; echo rc=$?
timeout 1200 python tools/autotune.py --ops tsmm --dtypes d,z --widths 16-64 --filter "c.get('impl', 0) in (2, 3)" --keep-better --time-budget 1000 > gpurun_out/autotune19b.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r19.json
python tools/gen_instances.py > /dev/null && python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build19.log 2>&1; echo build rc=$?
bash tools/ncu_run.sh r19 tsmttsm d 40x40 48x48 64x64
bash tools/ncu_run.sh r19 tsmm d 64x64
