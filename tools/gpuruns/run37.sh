# r37: inline-edge TSMTTSM -- parity, then autotune over the inline-edge candidates (keep-better against the stored autotune times) into a copy of the table
timeout 1500 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "inline_edge" > gpurun_out/pytest_ei37.log 2>&1; echo pytest rc=$?; tail -n 5 gpurun_out/pytest_ei37.log
cp tune/b200.json gpurun_out/b200_r37.json
timeout 1800 python tools/autotune.py --ops tsmttsm --dtypes d --widths 9,10,11,12,17,18,19,20,25,26,27,28,33,34,35,36,41,42,43,44,49,50,51,52,57,58,59,60 --filter "c.get('EI')" --keep-better --time-budget 1500 --out gpurun_out/b200_r37.json > gpurun_out/autotune37d.log 2>&1; echo autotune-d rc=$?
timeout 1800 python tools/autotune.py --ops tsmttsm --dtypes z --widths 9,10,11,12,17,18,19,20,25,26,27,28,33,34,35,36,41,42,43,44,49,50,51,52,57,58,59,60 --filter "c.get('EI')" --keep-better --time-budget 1500 --out gpurun_out/b200_r37.json > gpurun_out/autotune37z.log 2>&1; echo autotune-z rc=$?
