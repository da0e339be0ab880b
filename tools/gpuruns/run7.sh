timeout 2400 python tools/autotune.py --ops tsmttsm --dtypes d,z --widths 1-64 --time-budget 2200 > gpurun_out/autotune_tsmttsm.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_tsmttsm.json
tail -n 5 gpurun_out/autotune_tsmttsm.log
