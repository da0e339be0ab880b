timeout 2400 python tools/autotune.py --ops tsmm,tsmttsm --dtypes d,z --widths 1-64 --time-budget 2000 > gpurun_out/autotune9.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r9.json
tail -n 3 gpurun_out/autotune9.log
