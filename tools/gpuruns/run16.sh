timeout 2400 python tools/autotune.py --ops tsmttsm --dtypes d,z --widths 24-64 --time-budget 2000 > gpurun_out/autotune16.log 2>&1; echo rc=$?
cp tune/b200.json gpurun_out/b200_r16.json
